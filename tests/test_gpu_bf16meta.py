"""GPU vs oracle parity of NEXT-1, the paper's bf16 per-group metadata (
S:106-109; DESIGN reading 21), through actnn_quantize_bf16meta /
actnn_dequantize_bf16meta.  Bar as for the fp32 format: packed codes and the
metadata words bit-exact, dequantised values bit-exact.  Covers the single-pass
kernel (uniform widths), the warp-specialised mixed-path kernel, the generic
kernels (ragged D, unaligned input), both dequantiser metadata paths (TMA when
ng % 4 == 0, global loads otherwise), all widths, adversarial tensors and an
exhaustive full-size check."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2104_14129_b200 as A
    return A


@pytest.fixture(scope="module")
def W():
    from paper_2104_14129_b200 import workloads as W
    return W


def host(t):
    return t.detach().cpu().numpy()


def x_host(x):
    if x.dtype == torch.bfloat16:
        return host(x.contiguous().view(torch.int16)).view(np.uint16).reshape(x.shape[0], -1)
    return host(x).reshape(x.shape[0], -1)


def run_both(A, x, bits_np, seed, sample_base=0, two_pass=False):
    D = x[0].numel()
    bits_np = np.asarray(bits_np, np.uint8)
    bits = torch.from_numpy(bits_np).to(DEV)
    off = torch.from_numpy(O.offsets(bits_np, D)).to(DEV)
    gmin = gmax = None
    if two_pass:
        gmin, gmax, _ = A.group_stats(x)
    p = A.quantize(x, bits, off, seed, sample_base, gmin, gmax, meta="bf16")
    ref = O.quantize_bf16meta(x_host(x), bits_np, seed, sample_base, threads=8)
    return p, ref


def assert_equal(p, ref):
    packed, meta, off = ref
    nbytes = int(off[-1])
    got = host(p.packed[:nbytes])
    if not np.array_equal(got, packed):
        bad = np.nonzero(got != packed)[0]
        raise AssertionError(f"packed differs at {len(bad)} bytes, first {bad[:8]}")
    gm = host(p.meta).view(np.uint32)
    if not np.array_equal(gm, meta.ravel()):
        bad = np.nonzero(gm != meta.ravel())[0]
        raise AssertionError(f"meta differs at {len(bad)} groups, first {bad[:8]}")
    assert p.zmin is None and p.scale is None


def assert_dequant(A, p, ref, bits, N, D):
    packed, meta, _ = ref
    out = A.dequantize(p, out_dtype=torch.float32)
    exp = O.dequantize_bf16meta(packed, meta, bits, N, D)
    assert np.array_equal(host(out).reshape(N, D).view(np.uint32), exp.view(np.uint32))
    outb = A.dequantize(p, out_dtype=torch.bfloat16)
    expb = O.dequantize_bf16meta(packed, meta, bits, N, D, out_dtype=O.BF16)
    assert np.array_equal(host(outb.view(torch.int16)).reshape(N, D).view(np.uint16), expb)


@pytest.mark.parametrize("b", [1, 2, 4, 8, 3, 5, 6, 7])
def test_adversarial_all_widths_bf16meta(A, W, b):
    rng = np.random.default_rng(b)
    for name, xa in W.adversarial_tensors(rng).items():
        x = torch.from_numpy(xa).to(DEV)
        N, D = x.shape
        for two_pass in (False, True):
            p, ref = run_both(A, x, [b] * N, seed=4321 + b, sample_base=3, two_pass=two_pass)
            torch.cuda.synchronize()
            assert_equal(p, ref)
        assert_dequant(A, p, ref, [b] * N, N, D)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D", [256 * 70, 256 * 33, 1024])
def test_mixed_widths_multi_tile_bf16meta(A, W, dtype, D):
    """Widths 1,2,4,8 across samples, several units per sample, a ragged unit
    tail (ng = 70, 33: the dequantiser loads metadata without TMA when
    ng % 4 != 0), both compress kernels."""
    act = W.Act("t", D // 256, 16, 16, False)
    x = W.synth_activation(act, 8, 7, "f32" if dtype == torch.float32 else "bf16", DEV)
    bits = [1, 2, 4, 8, 8, 4, 2, 1]
    for two_pass in (False, True):
        p, ref = run_both(A, x, bits, seed=17, sample_base=100, two_pass=two_pass)
        torch.cuda.synchronize()
        assert_equal(p, ref)
    assert_dequant(A, p, ref, bits, 8, D)


@pytest.mark.parametrize("D", [7, 257, 700, 256 * 5 + 3])
def test_ragged_generic_bf16meta(A, D):
    rng = np.random.default_rng(D)
    xa = (rng.standard_normal((5, D)) * np.exp(rng.standard_normal((5, 1)))).astype(np.float32)
    x = torch.from_numpy(xa).to(DEV)
    bits = [1, 2, 4, 8, 3]
    for two_pass in (False, True):
        p, ref = run_both(A, x, bits, seed=2, sample_base=9, two_pass=two_pass)
        torch.cuda.synchronize()
        assert_equal(p, ref)
    assert_dequant(A, p, ref, bits, 5, D)


def test_unaligned_input_bf16meta(A):
    rng = np.random.default_rng(1)
    base = torch.from_numpy(rng.standard_normal(4 * 1024 + 1).astype(np.float32)).to(DEV)
    x = base[1:].view(4, 1024)
    p, ref = run_both(A, x, [2, 2, 4, 8], seed=3)
    torch.cuda.synchronize()
    assert_equal(p, ref)


@pytest.mark.parametrize("avg", [2.0, 1.25])
def test_compress_bf16meta_end_to_end(A, W, avg):
    """compress(avg_bits, meta='bf16'): stats -> allocation -> ws kernel; the
    allocation is unchanged by the metadata format (it uses the exact ranges,
    P:547), the codes follow the bf16 contract."""
    act = W.resnet_activation_set(50)[20]
    x = W.synth_activation(act, 32, 20, "f32", DEV)
    p = A.compress(x, seed=555, avg_bits=avg, meta="bf16")
    out = A.decompress(p)
    torch.cuda.synchronize()
    xh = x_host(x)
    gmin, gmax = O.group_minmax(xh)
    bits = O.allocate_bits(O.sensitivity(gmin, gmax), int(avg * 32))
    assert np.array_equal(host(p.bits), bits)
    ref = O.quantize_bf16meta(xh, bits, 555, 0, threads=8)
    assert_equal(p, ref)
    exp = O.dequantize_bf16meta(ref[0], ref[1], bits, 32, act.D, threads=8)
    assert np.array_equal(host(out).reshape(32, -1).view(np.uint32), exp.view(np.uint32))


def test_full_size_c3_layer_bf16meta_exhaustive(A, W):
    """The largest C3 tensor at batch 256 (822 MB fp32, the bench's launch
    configuration) with bf16 metadata, exhaustively: the device allocation
    against the oracle's O3 + O11 + O12, every packed byte, every metadata word
    and every dequantised value against the oracle (all host threads); every
    output inside its group's stored [Z', Z' + R']."""
    import os
    threads = os.cpu_count() or 1
    wl = W.workload("c3")
    act = wl.acts[1]
    x = W.synth_activation(act, wl.N, 1, "f32", DEV)
    seed = W.quant_seed(1)
    p = A.compress(x, seed=seed, avg_bits=2.0, meta="bf16")
    out = A.decompress(p)
    torch.cuda.synchronize()
    D = act.D
    ng = D // 256
    xh = x_host(x)
    gmin, gmax = O.group_minmax(xh)
    bits = O.allocate_bits(O.sensitivity(gmin, gmax), int(2.0 * wl.N))
    assert np.array_equal(host(p.bits), bits)
    ref = O.quantize_bf16meta(xh, bits, seed, 0, threads=threads)
    assert_equal(p, ref)
    exp = O.dequantize_bf16meta(ref[0], ref[1], bits, wl.N, D, threads=threads)
    assert np.array_equal(host(out).reshape(wl.N, D).view(np.uint32), exp.view(np.uint32))
    del exp, xh
    meta = host(p.meta).view(np.uint32)
    Z, R = O.meta_fields(meta.reshape(wl.N, ng))
    lo = torch.from_numpy(Z).to(DEV).view(wl.N, ng, 1)
    Rt = torch.from_numpy(R).to(DEV).view(wl.N, ng, 1)
    o = out.view(wl.N, ng, 256)
    # h_hat = fmaf(code, RN(R'/B), Z') >= Z' exactly; <= Z' + R' up to the two
    # roundings (|Z'| + R') 2^-23
    assert bool((o >= lo).all())
    assert bool((o <= lo + Rt + (lo.abs() + Rt) * 2 ** -22 + 1e-38).all())
