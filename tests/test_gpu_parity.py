"""GPU (CUDA path through the C ABI) vs CPU oracle parity.

Bar (BASELINE.json north_star): packed codes, zero points
and scales bit-exact; dequantised values bit-exact too (ACTNN-Q v1 makes
dequantisation one fmaf), which implies the north_star's 1e-6 * R guard;
allocator bits and offsets bit-exact.  Inputs come from
paper_2104_14129_b200.workloads (seeded, shared by both sides).
"""
import json
import os
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


DEV = "cuda:0"


def host(t):
    return t.detach().cpu().numpy()


def x_host(x):
    """fp32 -> float32 array; bf16 -> uint16 bit patterns (oracle input)."""
    if x.dtype == torch.bfloat16:
        return host(x.contiguous().view(torch.int16)).view(np.uint16).reshape(x.shape[0], -1)
    return host(x).reshape(x.shape[0], -1)


def assert_packed_equal(p, ref, N):
    packed, zmin, scale, off = ref
    off_g = host(p.off)
    assert np.array_equal(off_g - off_g[0], off), "offsets"
    nbytes = int(off[-1])
    got = host(p.packed[:nbytes])
    if not np.array_equal(got, packed):
        bad = np.nonzero(got != packed)[0]
        raise AssertionError(f"packed differs at {len(bad)} bytes, first {bad[:8]}")
    assert np.array_equal(host(p.zmin).view(np.uint32), zmin.ravel().view(np.uint32)), "zmin"
    assert np.array_equal(host(p.scale).view(np.uint32), scale.ravel().view(np.uint32)), "scale"


def run_both(A, x, bits_np, seed, sample_base=0, two_pass=False, threads=8):
    N = x.shape[0]
    D = x[0].numel()
    bits = torch.from_numpy(np.asarray(bits_np, np.uint8)).to(DEV)
    off = torch.from_numpy(O.offsets(np.asarray(bits_np, np.uint8), D)).to(DEV)
    gmin = gmax = None
    if two_pass:
        gmin, gmax, _ = A.group_stats(x)
    p = A.quantize(x, bits, off, seed, sample_base, gmin, gmax)
    ref = O.quantize(x_host(x), np.asarray(bits_np, np.uint8), seed, sample_base, threads=threads)
    return p, ref


# ----------------------------------------------------------------------------- C1 golden
def test_c1_golden(A, W):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c1.json")))
    x = torch.from_numpy(W.c1_tensor()).to(DEV)
    for two_pass in (False, True):
        if two_pass:
            gmin, gmax, _ = A.group_stats(x)
            bits, off = A.uniform_bits(4, 1024, 2, DEV)
            p = A.quantize(x, bits, off, 42, 0, gmin, gmax)
        else:
            p = A.compress(x, seed=42, bits=2)
        torch.cuda.synchronize()
        assert host(p.packed[:1024]).tobytes().hex() == g["packed_hex"]
        assert host(p.zmin).view(np.uint32).tolist() == g["zmin_bits"]
        assert host(p.scale).view(np.uint32).tolist() == g["scale_bits"]
        out = A.decompress(p)
        assert hashlib.sha256(host(out).tobytes()).hexdigest() == g["dequant_sha256"]


# ----------------------------------------------------------------------------- quantiser
@pytest.mark.parametrize("b", [1, 2, 4, 8, 3, 5, 6, 7])
def test_adversarial_all_widths(A, W, b):
    rng = np.random.default_rng(b)
    for name, xa in W.adversarial_tensors(rng).items():
        x = torch.from_numpy(xa).to(DEV)
        for two_pass in (False, True):
            p, ref = run_both(A, x, [b] * x.shape[0], seed=1234 + b, sample_base=5,
                              two_pass=two_pass)
            torch.cuda.synchronize()
            assert_packed_equal(p, ref, x.shape[0])
        out = A.dequantize(p)
        exp = O.dequantize(*ref[:3], np.full(x.shape[0], b, np.uint8), x.shape[0], x.shape[1])
        assert np.array_equal(host(out).view(np.uint32), exp.view(np.uint32)), name
        outb = A.dequantize(p, out_dtype=torch.bfloat16)
        expb = O.dequantize(*ref[:3], np.full(x.shape[0], b, np.uint8), x.shape[0], x.shape[1],
                            out_dtype=O.BF16)
        assert np.array_equal(host(outb.view(torch.int16)).view(np.uint16), expb), name


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D", [256 * 70, 256 * 33, 1024])
def test_mixed_widths_multi_tile(A, W, dtype, D):
    """Per-sample widths cycling 1,2,4,8 over several units and a ragged unit
    tail (ng = 70 -> 17 full 4-group units + one of 2)."""
    act = W.Act("t", D // 256, 16, 16, False)
    x = W.synth_activation(act, 8, 3, "f32" if dtype == torch.float32 else "bf16", DEV)
    bits = [1, 2, 4, 8, 8, 4, 2, 1]
    for two_pass in (False, True):
        p, ref = run_both(A, x, bits, seed=99, sample_base=1000, two_pass=two_pass)
        torch.cuda.synchronize()
        assert_packed_equal(p, ref, 8)
    out = A.dequantize(p)
    exp = O.dequantize(*ref[:3], np.array(bits, np.uint8), 8, D,
                       out_dtype=O.F32 if dtype == torch.float32 else O.BF16)
    got = host(out.view(torch.int16)).view(np.uint16) if dtype == torch.bfloat16 else host(out)
    assert np.array_equal(got.view(exp.dtype), exp)


@pytest.mark.parametrize("D", [1, 7, 255, 257, 700, 1000, 256 * 5 + 3])
def test_ragged_and_generic_path(A, D):
    """D % 256 != 0 takes the generic kernels (ragged last group)."""
    rng = np.random.default_rng(D)
    xa = (rng.standard_normal((5, D)) * np.exp(rng.standard_normal((5, 1)))).astype(np.float32)
    x = torch.from_numpy(xa).to(DEV)
    bits = [1, 2, 4, 8, 3]
    for two_pass in (False, True):
        p, ref = run_both(A, x, bits, seed=5, sample_base=2, two_pass=two_pass)
        torch.cuda.synchronize()
        assert_packed_equal(p, ref, 5)
    out = A.dequantize(p)
    exp = O.dequantize(*ref[:3], np.array(bits, np.uint8), 5, D)
    assert np.array_equal(host(out), exp)


def test_unaligned_input_generic_path(A):
    """A view starting 1 element into an allocation is not 32 B aligned."""
    rng = np.random.default_rng(0)
    base = torch.from_numpy(rng.standard_normal(4 * 1024 + 1).astype(np.float32)).to(DEV)
    x = base[1:].view(4, 1024)
    p, ref = run_both(A, x, [2, 2, 4, 8], seed=3)
    torch.cuda.synchronize()
    assert_packed_equal(p, ref, 4)


def test_empty_problem(A):
    x = torch.empty(0, 1024, device=DEV)
    p = A.compress(x, seed=1, bits=2)
    assert A.decompress(p).shape == (0, 1024)


# ----------------------------------------------------------------------------- stats
@pytest.mark.parametrize("D", [256 * 70, 256 * 3136, 700])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_group_stats_bit_exact(A, W, D, dtype):
    act = W.Act("t", 1, 1, D, True) if D % 256 else W.Act("t", D // 256, 16, 16, True)
    if D % 256:
        x = torch.from_numpy(np.random.default_rng(D).standard_normal((6, D)).astype(np.float32))
        x = x.to(DEV) if dtype == "f32" else x.to(torch.bfloat16).to(DEV)
    else:
        x = W.synth_activation(act, 6, 11, dtype, DEV)
    gmin, gmax, S = A.group_stats(x)
    torch.cuda.synchronize()
    omin, omax = O.group_minmax(x_host(x))
    assert np.array_equal(host(gmin).view(np.uint32), omin.ravel().view(np.uint32))
    assert np.array_equal(host(gmax).view(np.uint32), omax.ravel().view(np.uint32))
    assert np.array_equal(host(S).view(np.uint64), O.sensitivity(omin, omax).view(np.uint64))


# ----------------------------------------------------------------------------- allocator
def _w_cases(rng):
    yield "lognormal", np.exp(2.0 * rng.standard_normal(256))
    yield "wide", 10 ** rng.uniform(-6, 6, 1000)
    yield "equal", np.ones(300)
    yield "zeros", np.concatenate([np.zeros(50), np.exp(rng.standard_normal(50))])
    w = np.exp(rng.standard_normal(512))
    w[::3] = w[0]                              # many exact ties across samples
    yield "ties", w
    yield "n1023", np.exp(2.0 * rng.standard_normal(1023))   # K2 from global memory
    yield "n1024", np.exp(2.0 * rng.standard_normal(1024))   # K2 keys in shared memory
    yield "n4096", np.exp(rng.standard_normal(4096))
    yield "n20000", np.exp(3 * rng.standard_normal(20000))
    # K2 stages the sample weights in shared memory up to 24576 samples; above
    # that it reads them from global memory (both kernels, both tie paths)
    yield "n24576", np.exp(rng.standard_normal(24576))
    yield "n30000", np.exp(3 * rng.standard_normal(30000))
    yield "equal_n30000", np.ones(30000)
    yield "single", np.array([3.0])


@pytest.mark.parametrize("mask", [0x116, 0x1FE, 0x114, 0x100])
def test_allocate_matches_oracle_heap(A, mask):
    rng = np.random.default_rng(mask)
    levels = [b for b in range(8, 0, -1) if mask & (1 << b)]
    for name, w in _w_cases(rng):
        N = len(w)
        S = torch.from_numpy(w.astype(np.float64)).to(DEV)
        budgets = {N * levels[-1], N * levels[0], N * levels[0] + 7, int(1.25 * N), 2 * N,
                   int(3.3 * N), N * levels[-1] + 1}
        for budget in sorted(budgets):
            if budget < N * levels[-1]:
                continue
            bits, off = A.allocate_bits(S, budget, 256 * 98, mask)
            torch.cuda.synchronize()
            ref = O.allocate_bits(w, budget, mask)
            got = host(bits)
            assert np.array_equal(got, ref), (name, budget, np.nonzero(got != ref)[0][:5])
            assert np.array_equal(host(off), O.offsets(ref, 256 * 98)), (name, budget)


def test_allocate_with_gscale(A):
    rng = np.random.default_rng(9)
    S = np.exp(rng.standard_normal(777))
    gs = np.exp(rng.standard_normal(777))
    bits, _ = A.allocate_bits(torch.from_numpy(S).to(DEV), 1000, 1024,
                              gscale=torch.from_numpy(gs).to(DEV))
    ref = O.allocate_bits(S * gs, 1000)
    assert np.array_equal(host(bits), ref)


def test_allocate_infeasible_raises(A):
    with pytest.raises(A.ActnnError):
        A.allocate_bits(torch.ones(10, dtype=torch.float64, device=DEV), 9, 1024)


# ----------------------------------------------------------------------------- mixed path
@pytest.mark.parametrize("avg", [2.0, 1.25])
def test_mixed_path_end_to_end(A, W, avg):
    """stats -> allocate -> quantize(with stats) == oracle's sharded driver at k=1."""
    act = W.resnet_activation_set(50)[20]
    x = W.synth_activation(act, 32, 20, "f32", DEV)
    p = A.compress(x, seed=777, avg_bits=avg)
    torch.cuda.synchronize()
    packed, zmin, scale, bits = O.sharded_quantize(x_host(x), 1, avg, 777, threads=8)[0]
    assert np.array_equal(host(p.bits), bits)
    assert_packed_equal(p, (packed, zmin, scale, O.offsets(bits, act.D)), 32)


@pytest.mark.parametrize("k", [2, 4])
def test_virtual_ranks_equal_one_rank(A, W, k):
    """SURVEY §4 'virtual ranks': k batch slices on one GPU, S written into a
    zero-padded global vector per slice and summed (the all-reduce), global
    allocation, per-slice quantize with sample_base: the concatenation equals
    the single-rank output byte for byte, and the oracle's O13."""
    act = W.resnet_activation_set(50)[30]
    N = 16
    x = W.synth_activation(act, N, 30, "f32", DEV)
    one = A.compress(x, seed=4242, avg_bits=2.0)
    n_loc = N // k
    parts = []
    for r in range(k):
        xs = x[r * n_loc:(r + 1) * n_loc]

        def fake_allreduce(S_local, r=r):
            tot = torch.zeros_like(S_local)
            for q in range(k):
                Sq = torch.zeros_like(S_local)
                A.group_stats(x[q * n_loc:(q + 1) * n_loc], sens_out=Sq[q * n_loc:(q + 1) * n_loc])
                tot += Sq
            return tot

        parts.append(A.compress(xs, seed=4242, avg_bits=2.0, sample_base=r * n_loc,
                                sens_allreduce=fake_allreduce, n_total=N))
    torch.cuda.synchronize()
    cat_bits = np.concatenate([host(p.bits) for p in parts])
    assert np.array_equal(cat_bits, host(one.bits))
    cat_packed = np.concatenate([host(p.packed[:int(host(p.off)[-1] - host(p.off)[0])])
                                 for p in parts])
    one_bytes = host(one.packed[:int(host(one.off)[-1])])
    assert np.array_equal(cat_packed, one_bytes)
    assert np.array_equal(np.concatenate([host(p.zmin) for p in parts]), host(one.zmin))
    ref = O.sharded_quantize(x_host(x), k, 2.0, 4242, threads=8)
    assert np.array_equal(np.concatenate([r_[0] for r_ in ref]), one_bytes)


# ----------------------------------------------------------------------------- full size
def _sample_groups(rng, N, ng, k):
    gs = set()
    gs.update([(0, 0), (N - 1, ng - 1), (N // 2, ng // 2)])
    while len(gs) < k:
        gs.add((int(rng.integers(N)), int(rng.integers(ng))))
    return sorted(gs)


def _check_sampled_groups(A, x, p, seed, sample_base, samples, out=None):
    N = x.shape[0]
    D = x[0].numel()
    ng = -(-D // 256)
    bits = host(p.bits)
    off = host(p.off)
    for (n, i) in samples:
        b = int(bits[n])
        h = x[n].reshape(-1)[i * 256:(i + 1) * 256]
        hh = x_host(h.reshape(1, -1))[0]
        if hh.dtype == np.uint16:
            hh = (hh.astype(np.uint32) << 16).view(np.float32)
        e0 = (sample_base + n) * D + i * 256
        seg, z, s = O.quantize_group(hh, b, seed, e0)
        start = int(off[n] - off[0]) + i * 32 * b
        got = host(p.packed[start:start + 32 * b])
        assert np.array_equal(got, seg), (n, i, b)
        assert host(p.zmin[n * ng + i]).view(np.uint32) == np.float32(z).view(np.uint32)
        assert host(p.scale[n * ng + i]).view(np.uint32) == np.float32(s).view(np.uint32)
        if out is not None:
            _, vals = O.dequantize_group(seg, 256, b, z, s)
            got_o = host(out[n].reshape(-1)[i * 256:(i + 1) * 256].float())
            if out.dtype == torch.bfloat16:
                vals = torch.from_numpy(vals).to(torch.bfloat16).float().numpy()
            assert np.array_equal(got_o, vals), (n, i)


def test_full_size_c2_sampled(A, W):
    """C2 at full size (256 x 64 x 112 x 112 fp32, uniform 2-bit) in the launch
    configuration bench.py times; 256 sampled groups checked by the oracle one
    by one, plus global invariants."""
    wl = W.workload("c2")
    act = wl.acts[0]
    x = W.synth_activation(act, wl.N, 0, "f32", DEV)
    p = A.compress(x, seed=W.quant_seed(0), bits=2)
    out = A.decompress(p)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    _check_sampled_groups(A, x, p, W.quant_seed(0), 0, _sample_groups(rng, wl.N, 3136, 256), out)
    # |h_hat - h| <= one quantisation step everywhere (codes within [0, B])
    err = (out - x).abs().view(wl.N, 3136, 256).amax(dim=2)
    assert bool((err <= p.scale.view(wl.N, 3136) * (1 + 1e-6) + 1e-30).all())


@pytest.mark.parametrize("layer", [0, 1, 50, 106])
def test_full_size_c3_layer_sampled(A, W, layer):
    """C3 layers at full batch 256 through the mixed path: allocator bits
    bit-exact vs the oracle heap on the GPU's S; S itself and sampled groups
    checked against the oracle."""
    wl = W.workload("c3")
    act = wl.acts[layer]
    x = W.synth_activation(act, wl.N, layer, "f32", DEV)
    seed = W.quant_seed(layer)
    gmin, gmax, S = A.group_stats(x)
    bits, off = A.allocate_bits(S, int(2.0 * wl.N), act.D)
    p = A.quantize(x, bits, off, seed, 0, gmin, gmax)
    out = A.dequantize(p)
    torch.cuda.synchronize()
    Sh = host(S)
    assert np.array_equal(host(bits), O.allocate_bits(Sh, 512))
    rng = np.random.default_rng(layer)
    for n in rng.choice(wl.N, 4, replace=False):
        mn, mx = O.group_minmax(x_host(x[n:n + 1]))
        assert O.sensitivity(mn, mx)[0] == Sh[n]
    ng = -(-act.D // 256)
    _check_sampled_groups(A, x, p, seed, 0, _sample_groups(rng, wl.N, ng, 128), out)


def test_full_size_c4_layer_bf16_sampled(A, W):
    """C4's largest layer (ResNet-152 stem bn1 input, batch 1024, bf16, 1.25 bits)."""
    wl = W.workload("c4")
    act = wl.acts[1]
    x = W.synth_activation(act, wl.N, 1, "bf16", DEV)
    seed = W.quant_seed(1)
    p = A.compress(x, seed=seed, avg_bits=1.25)
    out = A.decompress(p)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    _check_sampled_groups(A, x, p, seed, 0, _sample_groups(rng, wl.N, act.D // 256, 128), out)
    assert int(host(p.bits).astype(np.int64).sum()) <= int(1.25 * wl.N)


def test_compress_sharded_one_rank_nccl(A, W):
    """dist.compress_sharded through a real (1-rank) NCCL group equals the
    unsharded call byte for byte."""
    import torch.distributed as dist
    from paper_2104_14129_b200 import dist as AD
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        act = W.resnet_activation_set(50)[12]
        x = W.synth_activation(act, 8, 12, "f32", DEV)
        a = AD.compress_sharded(x, 99, 2.0)
        b = A.compress(x, seed=99, avg_bits=2.0)
        torch.cuda.synchronize()
        nb = int(host(b.off)[-1])
        assert np.array_equal(host(a.packed[:nb]), host(b.packed[:nb]))
        assert np.array_equal(host(a.bits), host(b.bits))
    finally:
        dist.destroy_process_group()


def test_pipelined_step_graph_with_nccl_gather(A, W):
    """The pipelined step with the NCCL exchange of S (1-rank group) captured in
    a CUDA graph: replays equal the eager step byte for byte (the multi-GPU
    bench replays this graph).  Runs in a fresh process: a process group
    created after another one was destroyed in the same process does not
    replay its captured collectives (observed in this suite)."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "..", "tools",
                                                     "graph_nccl_check.py")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("sample_base", [524284, 524285, 2 ** 30])
@pytest.mark.parametrize("two_pass", [False, True])
def test_philox_counter_high_word(A, sample_base, two_pass):
    """Global element indices up to exactly 2^35 (524284: the last Philox
    counter is 2^32 - 1, fast kernels with the 32-bit-counter Philox) and past
    it (counter high word non-zero: the generic kernel carries the 64-bit
    counter); both equal the oracle."""
    D = 65536
    g = torch.Generator(device=DEV).manual_seed(sample_base)
    x = torch.randn((4, D), generator=g, device=DEV)
    for bits in ([1, 2, 4, 8], [2, 2, 2, 2]):
        p, ref = run_both(A, x, bits, seed=77, sample_base=sample_base, two_pass=two_pass)
        assert_packed_equal(p, ref, 4)


def test_api_validates_caller_buffers(A):
    """caller-supplied buffers are checked (device, contiguity,
    dtype, size) before their pointers reach the C ABI."""
    x = torch.randn(4, 1024, device=DEV)
    p = A.compress(x, seed=1, bits=2)
    with pytest.raises(A.ActnnError):
        A.dequantize(p, out=torch.empty(4, 1000, device=DEV))            # too small
    with pytest.raises(A.ActnnError):
        A.dequantize(p, out=torch.empty(4, 2048, device=DEV)[:, ::2])    # strided
    with pytest.raises(A.ActnnError):
        A.dequantize(p, out=torch.empty(4, 1024, dtype=torch.float16, device=DEV))
    bits, off = A.uniform_bits(4, 1024, 2, DEV)
    with pytest.raises(A.ActnnError):
        A.quantize(x, bits, off.to(torch.int32), 1)
    with pytest.raises(A.ActnnError):
        A.quantize(x, bits[:3], off, 1)
    gmin, gmax, _ = A.group_stats(x)
    with pytest.raises(A.ActnnError):
        A.quantize(x, bits, off, 1, 0, gmin, None)
    with pytest.raises(A.ActnnError):
        A.quantize(x, bits, off, 1, 0, gmin[:-1], gmax)
    S = torch.ones(8, dtype=torch.float64, device=DEV)
    with pytest.raises(A.ActnnError):
        A.allocate_bits(S, 16, 1024, gscale=torch.ones(8, device=DEV))   # fp32 gscale
    with pytest.raises(A.ActnnError):
        A.gradmag_gather(torch.ones(10, dtype=torch.float64, device=DEV),
                         torch.zeros(3, dtype=torch.int32, device=DEV))
    mask, _ = A.relu_pack(x)
    with pytest.raises(A.ActnnError):
        A.relu_backward(mask[:10], x)
    x4 = torch.randn(2, 3, 16, 16, device=DEV)
    y, idx = A.maxpool2d(x4, 3, 2, 1)
    with pytest.raises(A.ActnnError):
        A.maxpool2d_backward(idx, y[..., :-1].contiguous(), 16, 16, 3, 2, 1)
    with pytest.raises(A.ActnnError):
        A.maxpool2d_backward(idx.to(torch.int32), y, 16, 16, 3, 2, 1)
    # the checks reject nothing valid
    out = A.dequantize(p, out=torch.empty(4, 1024, device=DEV))
    assert A.maxpool2d_backward(idx, y, 16, 16, 3, 2, 1).shape == x4.shape
    assert p.nbytes() < p.capacity_bytes()
    assert p.payload_bytes() == 4 * 4 * 32 * 2
