"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/actnn.h declares, and its host-side argument validation
returns the documented status without launching anything."""
import ctypes
import subprocess

import numpy as np
import pytest

from paper_2104_14129_b200 import _lib

OK, INVALID, UNSUPPORTED, BUDGET = 0, -1, -2, -3


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_exports_every_header_symbol(lib):
    names = _lib.header_symbols()
    assert len(names) == 21
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(names) <= exported


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_sizes(lib):
    assert lib.actnn_abi_version() == 1
    assert lib.actnn_workspace_bytes(0, 4, 1024, 256) == 4 * 1 * 8 + 8
    assert lib.actnn_workspace_bytes(0, 2, 256 * 33, 256) == 2 * 2 * 8 + 8
    assert lib.actnn_workspace_bytes(1, 4, 1024, 256) == 0
    assert lib.actnn_packed_bytes(4, 1024, 256, None) == 4 * 4 * 256
    bits = np.array([1, 2, 4, 8], np.uint8)
    p = bits.ctypes.data_as(ctypes.c_void_p)
    assert lib.actnn_packed_bytes(4, 1000, 256, p) == 15 * 4 * 32
    bad = np.array([0, 9], np.uint8)
    assert lib.actnn_packed_bytes(2, 256, 256, bad.ctypes.data_as(ctypes.c_void_p)) == -1


def _msg(lib):
    return lib.actnn_last_error().decode()


def test_quantize_host_validation(lib):
    d = ctypes.c_void_p(0x1000)  # never dereferenced: validation fails first
    q = lib.actnn_quantize
    assert q(None, 0, 4, 1024, 256, d, d, 1, 0, None, None, d, d, d, None) == INVALID
    assert "null" in _msg(lib)
    assert q(d, 0, 4, 1024, 128, d, d, 1, 0, None, None, d, d, d, None) == UNSUPPORTED
    assert q(d, 0, -1, 1024, 256, d, d, 1, 0, None, None, d, d, d, None) == INVALID
    assert q(d, 7, 4, 1024, 256, d, d, 1, 0, None, None, d, d, d, None) == INVALID
    assert q(d, 0, 4, 1024, 256, d, d, 1, 0, d, None, d, d, d, None) == INVALID
    assert q(d, 0, 4, 1024, 256, d, d, 1, -5, None, None, d, d, d, None) == INVALID
    unal = ctypes.c_void_p(0x1008)
    assert q(d, 0, 4, 1024, 256, d, d, 1, 0, None, None, unal, d, d, None) == UNSUPPORTED
    assert q(ctypes.c_void_p(0x1002), 0, 4, 1024, 256, d, d, 1, 0, None, None, d, d, d,
             None) == INVALID
    # empty problems are valid no-ops
    assert q(None, 0, 0, 1024, 256, None, None, 1, 0, None, None, None, None, None, None) == OK
    assert q(None, 0, 4, 0, 256, None, None, 1, 0, None, None, None, None, None, None) == OK


def test_dequantize_and_stats_host_validation(lib):
    d = ctypes.c_void_p(0x1000)
    dq = lib.actnn_dequantize
    assert dq(None, d, d, d, d, 4, 1024, 256, d, 0, None) == INVALID
    assert dq(d, d, d, d, d, 4, 1024, 512, d, 0, None) == UNSUPPORTED
    assert dq(d, d, d, d, d, 4, 1024, 256, d, 3, None) == INVALID
    assert dq(None, None, None, None, None, 0, 1024, 256, None, 0, None) == OK
    gs = lib.actnn_group_stats
    assert gs(d, 0, 4, 1024, 256, d, d, d, d, 0, None) == INVALID   # workspace too small
    assert "workspace" in _msg(lib)
    assert gs(d, 0, 4, 1024, 256, d, None, d, d, 64, None) == INVALID
    assert gs(None, 0, 0, 1024, 256, None, None, None, None, 0, None) == OK


def test_bf16meta_host_validation(lib):
    """NEXT-1 entry points: the same host checks; meta replaces zmin/scale."""
    d = ctypes.c_void_p(0x1000)
    q = lib.actnn_quantize_bf16meta
    assert q(d, 0, 4, 1024, 256, d, d, 1, 0, None, None, d, None, None) == INVALID
    assert "null" in _msg(lib)
    assert q(d, 0, 4, 1024, 128, d, d, 1, 0, None, None, d, d, None) == UNSUPPORTED
    assert q(d, 0, 4, 1024, 256, d, d, 1, 0, None, None, d, ctypes.c_void_p(0x1002),
             None) == INVALID
    assert q(d, 0, 4, 1024, 256, d, d, 1, 0, None, None, ctypes.c_void_p(0x1008), d,
             None) == UNSUPPORTED
    assert q(None, 0, 0, 1024, 256, None, None, 1, 0, None, None, None, None, None) == OK
    dq = lib.actnn_dequantize_bf16meta
    assert dq(d, None, d, d, 4, 1024, 256, d, 0, None) == INVALID
    assert dq(d, d, d, d, 4, 1024, 256, d, 5, None) == INVALID
    assert dq(None, None, None, None, 0, 1024, 256, None, 0, None) == OK


def test_contexts_host_validation(lib):
    """NEXT-4 entry points: host checks (geometry, the 256-tap limit of the
    8-bit index, null pointers, empty problems)."""
    d = ctypes.c_void_p(0x1000)
    assert lib.actnn_relu_pack(d, 0, -1, d, None, None) == INVALID
    assert lib.actnn_relu_pack(None, 0, 10, d, None, None) == INVALID
    assert lib.actnn_relu_pack(None, 0, 0, None, None, None) == OK
    assert lib.actnn_relu_pack(ctypes.c_void_p(0x1002), 0, 10, d, None, None) == INVALID
    assert lib.actnn_relu_backward(d, None, 1, 10, d, None) == INVALID
    fw, bw = lib.actnn_maxpool2d_forward, lib.actnn_maxpool2d_backward
    geo = (3, 3, 2, 2, 1, 1, 1, 1)
    assert fw(d, 0, 4, 112, 112, *geo, None, d, None) == INVALID
    assert fw(d, 0, 4, 112, 112, 17, 16, 1, 1, 0, 0, 1, 1, d, d, None) == UNSUPPORTED
    assert "8-bit" in _msg(lib)
    assert fw(d, 0, 4, 112, 112, 3, 3, 0, 2, 1, 1, 1, 1, d, d, None) == INVALID  # stride 0
    assert fw(d, 0, 4, 112, 112, 3, 3, 2, 2, 2, 1, 1, 1, d, d, None) == INVALID  # pad > k/2
    assert fw(d, 0, 4, 2, 2, 5, 5, 1, 1, 0, 0, 1, 1, d, d, None) == INVALID      # empty output
    # dilation 2, padding 1, a 1-row input: the only window's taps (-1, 1) miss it
    assert fw(d, 0, 4, 1, 4, 2, 1, 1, 1, 1, 0, 2, 1, d, d, None) == UNSUPPORTED
    assert "padding" in _msg(lib)
    assert bw(d, d, 0, 4, 1, 4, 2, 1, 1, 1, 1, 0, 2, 1, d, None) == UNSUPPORTED
    assert fw(None, 0, 0, 112, 112, *geo, None, None, None) == OK
    assert bw(None, d, 0, 4, 112, 112, *geo, d, None) == INVALID


def test_allocate_host_validation(lib):
    d = ctypes.c_void_p(0x1000)
    al = lib.actnn_allocate_bits
    POW2 = 0x116
    assert al(d, None, 10, 9, POW2, 1024, 256, d, d, None, 0, None) == BUDGET
    assert "infeasible" in _msg(lib)
    assert al(d, None, 10, 40, 0x201, 1024, 256, d, d, None, 0, None) == INVALID
    assert al(d, None, 10, 40, 0, 1024, 256, d, d, None, 0, None) == INVALID
    assert al(None, None, 10, 40, POW2, 1024, 256, d, d, None, 0, None) == INVALID
    assert al(d, None, 10, 40, POW2, 1024, 100, d, d, None, 0, None) == UNSUPPORTED
    # unit-step mask: infeasible below N * 1
    assert al(d, None, 10, 9, 0x1FE, 1024, 256, d, d, None, 0, None) == BUDGET
    ub = lib.actnn_uniform_bits
    assert ub(4, 1024, 256, 0, d, d, None) == INVALID
    assert ub(4, 1024, 256, 9, d, d, None) == INVALID


def test_python_binding_refuses_cpu_tensors():
    torch = pytest.importorskip("torch")
    import paper_2104_14129_b200 as A
    with pytest.raises(A.ActnnError):
        A.quantize(torch.zeros(4, 1024), torch.zeros(4, dtype=torch.uint8),
                   torch.zeros(5, dtype=torch.int64), 0)


def test_plan_shard_without_exchange_is_refused():
    """A shard of a larger batch (n_total != N) cannot allocate without the
    exchange of S (the global S would stay all zeros)."""
    torch = pytest.importorskip("torch")
    from paper_2104_14129_b200.plan import ActivationSetPlan
    with pytest.raises(ValueError, match="gather"):
        ActivationSetPlan([torch.zeros(4, 1024)], [1], avg_bits=2.0, n_total=8, sample_base=4)


def test_adaptation_host_validation(lib):
    """NEXT-3 entry points: documented statuses before any launch."""
    d = ctypes.c_void_p(0x1000)
    D3 = (ctypes.c_int64 * 3)(10, 20, 30)
    assert lib.actnn_workspace_bytes(2, 4, 1024, 256) == 4 * 8 + 8
    assert lib.actnn_grad_sqnorm(None, 0, 4, 1024, 256, d, d, 64, None) == INVALID
    assert lib.actnn_grad_sqnorm(d, 0, 4, 1024, 128, d, d, 64, None) == UNSUPPORTED
    assert lib.actnn_grad_sqnorm(d, 0, 4, 1024, 256, d, d, 8, None) == INVALID  # small ws
    assert lib.actnn_grad_sqnorm(d, 0, 0, 1024, 256, None, None, 0, None) == OK
    assert lib.actnn_gradmag_ema(d, 4, 1.5, d, None) == INVALID
    assert lib.actnn_gradmag_ema(None, 0, 0.9, None, None) == OK
    assert lib.actnn_gradmag_gather(d, 0, d, 3, d, None) == INVALID
    assert lib.actnn_gradmag_scatter(d, 10, None, d, 3, None) == INVALID
    assert lib.actnn_allocate_layers_ws_bytes(3, 8, 0x116) >= 3 * 8 * 3 * 8
    assert lib.actnn_allocate_layers_ws_bytes(3, 8, 0) == 0
    al = lib.actnn_allocate_layers
    # infeasible: below sum_l D_l N * 1
    assert al(d, None, None, D3, 3, 2, 119, 0x116, d, d, d, 1 << 20, None) == BUDGET
    assert "infeasible" in _msg(lib)
    assert al(d, None, None, D3, 2000, 2, 10 ** 9, 0x116, d, d, d, 1 << 20, None) == UNSUPPORTED
    assert al(d, None, None, D3, 3, 2, 500, 0x3, d, d, d, 1 << 20, None) == INVALID  # mask
    bigD = (ctypes.c_int64 * 1)(1 << 25)
    assert al(d, None, None, bigD, 1, 2, 1 << 30, 0x116, d, d, d, 1 << 20, None) == UNSUPPORTED
    assert al(d, None, None, D3, 3, 2, 500, 0x116, d, d, d, 16, None) == INVALID  # small ws
    assert al(None, None, None, None, 0, 5, 0, 0x116, None, None, None, 0, None) == OK
