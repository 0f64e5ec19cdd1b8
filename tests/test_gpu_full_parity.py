"""Exhaustive GPU-vs-oracle parity at BASELINE.json's full sizes.

north_star: "bit-exact codes vs the oracle on every config"; SURVEY.md §8(d)
table D-1 asks for *full* parity on C2/C3 and "full, per layer, streamed" on
C4.  These tests run the step exactly as bench.py times it -- the same
ActivationSetPlan, the same plan.PipelinedStep (statistics / allocation /
quantisation / decompression streams) replayed from its captured CUDA graph --
and then compare EVERY output of EVERY tensor with the CPU oracle run from
the same host copy of the input (its own min/max, S_n, heap allocation,
quantiser and dequantiser):

  * S_n (fp64 bits), the per-sample widths and byte offsets;
  * every packed byte, every zmin / scale bit pattern;
  * every dequantised value (bit patterns; bf16 outputs as their bits).

C4's 311 tensors (91.5 GB of bf16 inputs) are compared one tensor at a time
(host memory holds one tensor); its decompression is checked with the same
per-tensor K4 launch the schedule issues, into a scratch buffer.

Also here: the kernel variants taken when N > 2048 samples (the per-sample
(bits, off) tables no longer fit shared memory: kCached = false) for the
single-pass, warp-specialised and dequantise kernels.
"""
import ctypes
import os
import threading
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
CORES = os.cpu_count() or 1


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


def out_bits(t, n_elems):
    """Dequantised outputs as raw bit patterns (u32 fp32 / u16 bf16)."""
    t = t[:n_elems]
    if t.dtype == torch.bfloat16:
        return host(t.view(torch.int16)).view(np.uint16)
    return host(t).view(np.uint32)


def oracle_minmax(xh):
    """O3 per sample slice on all host cores (the oracle call itself is
    single-threaded; ctypes releases the GIL)."""
    N = xh.shape[0]
    k = max(1, min(CORES, N))
    parts = [None] * k
    bounds = [(N * i // k, N * (i + 1) // k) for i in range(k)]

    def run(i):
        a, b = bounds[i]
        parts[i] = O.group_minmax(xh[a:b])

    ts = [threading.Thread(target=run, args=(i,)) for i in range(k)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))


def oracle_layer(xh, avg_bits, seed, out_dtype):
    """The whole hot path on the CPU for one tensor (O3, O11, O12, O5-O10)."""
    N, D = xh.shape
    gmin, gmax = oracle_minmax(xh)
    S = O.sensitivity(gmin, gmax)
    bits = O.allocate_bits(S, int(avg_bits * N))
    packed, zmin, scale, off = O.quantize(xh, bits, seed, 0, threads=CORES)
    out = O.dequantize(packed, zmin, scale, bits, N, D, out_dtype=out_dtype, threads=CORES)
    return S, bits, off, packed, zmin, scale, out


def compare_layer(i, L, ref, out_gpu_bits):
    S, bits, off, packed, zmin, scale, out = ref
    tag = f"tensor {i} [{L.N} x {L.D}]"
    assert np.array_equal(host(L.S[:L.N]).view(np.uint64), S.view(np.uint64)), tag + ": S_n"
    assert np.array_equal(host(L.bits[:L.N]), bits), tag + ": widths"
    off_g = host(L.off[:L.N + 1])
    assert np.array_equal(off_g - off_g[0], off), tag + ": offsets"
    nb = int(off[-1])
    got = host(L.packed[:nb])
    if not np.array_equal(got, packed):
        bad = np.nonzero(got != packed)[0]
        raise AssertionError(f"{tag}: {len(bad)} packed bytes differ, first at {bad[:8]}")
    assert np.array_equal(host(L.zmin).view(np.uint32), zmin.ravel().view(np.uint32)), tag
    assert np.array_equal(host(L.scale).view(np.uint32), scale.ravel().view(np.uint32)), tag
    exp = out.ravel().view(np.uint32 if out.dtype == np.float32 else np.uint16)
    if not np.array_equal(out_gpu_bits, exp):
        bad = np.nonzero(out_gpu_bits != exp)[0]
        raise AssertionError(f"{tag}: {len(bad)} dequantised values differ, first {bad[:8]}")


def build_step(A, W, wl, outs_per_layer):
    from paper_2104_14129_b200.plan import ActivationSetPlan, PipelinedStep
    xs = [W.synth_activation(a, wl.N, t, wl.dtype, DEV) for t, a in enumerate(wl.acts)]
    plan = ActivationSetPlan(xs, [W.quant_seed(t) for t in range(len(wl.acts))],
                             avg_bits=wl.avg_bits, level_mask=A.api.LEVELS_POW2)
    tdt = torch.float32 if wl.dtype == "f32" else torch.bfloat16
    if outs_per_layer:
        outs = [torch.empty(x.numel(), dtype=tdt, device=DEV) for x in xs]
    else:
        outs = [torch.empty(max(x.numel() for x in xs), dtype=tdt, device=DEV) for _ in range(3)]
    out_dt = A.api.F32 if wl.dtype == "f32" else A.api.BF16
    ps = PipelinedStep(plan, outs, out_dt)
    torch.cuda.set_stream(ps.stream)
    ps()                 # eager step
    ps.capture()         # graph capture + one replay
    for L in plan.layers:   # poison the step's outputs: the checked replay must rewrite them
        L.packed.fill_(0xA5)
        if L.zmin is not None:
            L.zmin.fill_(float("nan"))
            L.scale.fill_(float("nan"))
        L.bits.fill_(0)
        L.S.fill_(-1.0)
    for o in outs:
        o.fill_(float("nan"))
    ps()                 # the replay whose outputs are checked
    torch.cuda.synchronize()
    return xs, plan, ps, outs, out_dt


def test_c3_whole_step_exhaustive(A, W):
    """C3 (ResNet-50 set, 107 tensors, batch 256, fp32, mixed {1,2,4,8} at 2.0
    bits): the graph-replayed bench step, every output of every tensor."""
    torch.cuda.empty_cache()
    wl = W.workload("c3")
    xs, plan, ps, outs, _ = build_step(A, W, wl, outs_per_layer=True)
    t0 = time.time()
    for i, (x, L) in enumerate(zip(xs, plan.layers)):
        xh = x_host(x)
        ref = oracle_layer(xh, wl.avg_bits, W.quant_seed(i), O.F32)
        compare_layer(i, L, ref, out_bits(outs[i], x.numel()))
    print(f"C3: {len(xs)} tensors, {sum(x.numel() for x in xs)} elements compared "
          f"in {time.time() - t0:.1f} s on {CORES} cores")
    del xs, plan, ps, outs
    torch.cuda.set_stream(torch.cuda.default_stream())
    torch.cuda.empty_cache()


def test_c4_whole_step_exhaustive_streamed(A, W):
    """C4 (ResNet-152 set, 311 tensors, batch 1024, bf16, 1.25 bits): the
    graph-replayed bench step; then, tensor by tensor, the compressed outputs
    against the oracle and the tensor's K4 launch (as the schedule issues it)
    into a scratch buffer against the oracle's dequantisation."""
    torch.cuda.empty_cache()
    wl = W.workload("c4")
    xs, plan, ps, outs, out_dt = build_step(A, W, wl, outs_per_layer=False)
    scratch = outs[0]
    t0 = time.time()
    for i, (x, L) in enumerate(zip(xs, plan.layers)):
        plan.decompress_layer(i, scratch, out_dt, ctypes.c_void_p(ps.stream.cuda_stream))
        torch.cuda.synchronize()
        xh = x_host(x)
        ref = oracle_layer(xh, wl.avg_bits, W.quant_seed(i), O.BF16)
        compare_layer(i, L, ref, out_bits(scratch, x.numel()))
    print(f"C4: {len(xs)} tensors, {sum(x.numel() for x in xs)} elements compared "
          f"in {time.time() - t0:.1f} s on {CORES} cores")
    del xs, plan, ps, outs
    torch.cuda.set_stream(torch.cuda.default_stream())
    torch.cuda.empty_cache()


def test_c2_full_exhaustive(A, W):
    """C2 (one 822 MB fp32 tensor, uniform 2-bit, single pass): every byte and
    every dequantised value."""
    wl = W.workload("c2")
    x = W.synth_activation(wl.acts[0], wl.N, 0, "f32", DEV)
    seed = W.quant_seed(0)
    p = A.compress(x, seed=seed, bits=2)
    out = A.decompress(p)
    torch.cuda.synchronize()
    xh = x_host(x)
    packed, zmin, scale, off = O.quantize(xh, 2, seed, 0, threads=CORES)
    assert np.array_equal(host(p.packed[:int(off[-1])]), packed)
    assert np.array_equal(host(p.zmin).view(np.uint32), zmin.ravel().view(np.uint32))
    assert np.array_equal(host(p.scale).view(np.uint32), scale.ravel().view(np.uint32))
    exp = O.dequantize(packed, zmin, scale, 2, wl.N, wl.acts[0].D, threads=CORES)
    assert np.array_equal(host(out).reshape(wl.N, -1).view(np.uint32), exp.view(np.uint32))


# ------------------------------------------------------------------ N > 2048 variants
def _run_large_n(A, x, bits_np, seed, sample_base, two_pass, meta="f32"):
    N, D = x.shape[0], x[0].numel()
    bits = torch.from_numpy(bits_np).to(DEV)
    off = torch.from_numpy(O.offsets(bits_np, D)).to(DEV)
    gmin = gmax = None
    if two_pass:
        gmin, gmax, _ = A.group_stats(x)
    p = A.quantize(x, bits, off, seed, sample_base, gmin, gmax, meta=meta)
    torch.cuda.synchronize()
    return p


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D", [1024, 256 * 5, 256 * 9])
def test_uncached_variants_n4100(A, W, dtype, D):
    """N = 4100 > 2048: the quantisers (single pass and warp-specialised) and
    the dequantiser read (bits, off) from global memory (kCached = false);
    ng = 4 (metadata staged by TMA in K4) and ng = 5, 9 (ragged 4-group units,
    metadata read directly).  Widths cycle through {1, 2, 4, 8} and 3/5/6/7."""
    N = 4100
    act = W.Act("t", D // 256, 16, 16, True)
    x = W.synth_activation(act, N, 77, "f32" if dtype == torch.float32 else "bf16", DEV)
    cyc = np.array([1, 2, 4, 8, 3, 5, 6, 7, 2, 1], np.uint8)
    bits_np = cyc[np.arange(N) % len(cyc)]
    xh = x_host(x)
    ref = O.quantize(xh, bits_np, 4242, 17, threads=CORES)
    exp = O.dequantize(*ref[:3], bits_np, N, D, out_dtype=O.F32, threads=CORES)
    expb = O.dequantize(*ref[:3], bits_np, N, D, out_dtype=O.BF16, threads=CORES)
    for two_pass in (False, True):
        p = _run_large_n(A, x, bits_np, 4242, 17, two_pass)
        nb = int(ref[3][-1])
        assert np.array_equal(host(p.packed[:nb]), ref[0]), ("packed", two_pass)
        assert np.array_equal(host(p.zmin).view(np.uint32), ref[1].ravel().view(np.uint32))
        assert np.array_equal(host(p.scale).view(np.uint32), ref[2].ravel().view(np.uint32))
        out = A.dequantize(p, out_dtype=torch.float32)
        outb = A.dequantize(p, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        assert np.array_equal(host(out).reshape(N, D).view(np.uint32), exp.view(np.uint32))
        assert np.array_equal(host(outb.view(torch.int16)).view(np.uint16).reshape(N, D), expb)
    # NEXT-1 metadata words through the same uncached kernels
    refm = O.quantize_bf16meta(xh, bits_np, 99, 0, threads=CORES)
    for two_pass in (False, True):
        p = _run_large_n(A, x, bits_np, 99, 0, two_pass, meta="bf16")
        assert np.array_equal(host(p.packed[:int(refm[2][-1])]), refm[0])
        assert np.array_equal(host(p.meta).view(np.uint32), refm[1].ravel())
        out = A.dequantize(p, out_dtype=torch.float32)
        torch.cuda.synchronize()
        expm = O.dequantize_bf16meta(refm[0], refm[1], bits_np, N, D, threads=CORES)
        assert np.array_equal(host(out).reshape(N, D).view(np.uint32), expm.view(np.uint32))


def test_uncached_mixed_path_n4096_end_to_end(A, W):
    """stats -> allocation -> quantise at N = 4096 (C5's batch on one GPU, one
    ResNet-152 tensor shape): widths from the device allocator, bytes equal to
    the oracle's O12 + O5-O9."""
    wl = W.workload("c5")
    act = wl.acts[250]
    x = W.synth_activation(act, wl.N, 250, "bf16", DEV)
    p = A.compress(x, seed=W.quant_seed(250), avg_bits=1.25)
    out = A.decompress(p)
    torch.cuda.synchronize()
    xh = x_host(x)
    S, bits, off, packed, zmin, scale, oout = oracle_layer(xh, 1.25, W.quant_seed(250), O.BF16)
    assert np.array_equal(host(p.bits), bits)
    assert np.array_equal(host(p.packed[:int(off[-1])]), packed)
    assert np.array_equal(host(p.zmin).view(np.uint32), zmin.ravel().view(np.uint32))
    assert np.array_equal(out_bits(out.reshape(-1), out.numel()), oout.ravel())


@pytest.mark.parametrize("N,D", [(4100, 256 * 49), (4100, 256 * 48), (2048, 256 * 100),
                                 (2000, 256 * 101)])
def test_tma_store_dequantize_large_fp32(A, W, N, D):
    """fp32 outputs of >= 192 MB take the TMA-store K4 (shared-memory staging,
    cp.async.bulk shared -> global): cached / uncached (bits, off) tables,
    metadata staged (ng % 4 == 0) or read directly, ragged 4-group tails, all
    widths; every dequantised value against the oracle."""
    act = W.Act("t", D // 256, 16, 16, False)
    x = W.synth_activation(act, N, 91, "f32", DEV)
    assert x.numel() * 4 >= 192 << 20
    cyc = np.array([2, 1, 4, 8, 3, 5, 6, 7, 1, 2], np.uint8)
    bits_np = cyc[np.arange(N) % len(cyc)]
    p = _run_large_n(A, x, bits_np, 5150, 3, two_pass=True)
    out = A.dequantize(p, out_dtype=torch.float32)
    torch.cuda.synchronize()
    xh = x_host(x)
    ref = O.quantize(xh, bits_np, 5150, 3, threads=CORES)
    assert np.array_equal(host(p.packed[:int(ref[3][-1])]), ref[0])
    exp = O.dequantize(*ref[:3], bits_np, N, D, out_dtype=O.F32, threads=CORES)
    got = host(out).reshape(N, D).view(np.uint32)
    if not np.array_equal(got, exp.view(np.uint32)):
        bad = np.argwhere(got != exp.view(np.uint32))
        raise AssertionError(f"{len(bad)} values differ, first {bad[:4].tolist()}")


def test_c5_eight_virtual_ranks_plan_path(A, W):
    """"k-rank == 1-rank plus rank 0's shard".  One
    C5 tensor (ResNet-152 layer4.1.conv2 input shape, batch 4096, bf16, avg 1.25
    bits) split over k = 8 virtual ranks of 512 samples, each driven through
    the product's multi-rank path (ActivationSetPlan with n_total / sample_base
    and an exchange closure, PipelinedStep) on one GPU.  The closure delivers
    every rank's S_n (each rank's own slice is checked against what its stats
    kernel wrote); every rank's widths, packed bytes, zmin / scale and
    dequantised values must equal the oracle's sharded driver O13 for that rank
    (P:541-566 global greedy, P:491-508 per-group quantisation)."""
    from paper_2104_14129_b200.plan import ActivationSetPlan, PipelinedStep
    wl = W.workload("c5")
    t = 300
    act = wl.acts[t]
    N, k = wl.N, 8
    n_loc = N // k
    x = W.synth_activation(act, N, t, "bf16", DEV)
    S_all = torch.zeros(N, dtype=torch.float64, device=DEV)
    for r in range(k):
        A.group_stats(x[r * n_loc:(r + 1) * n_loc], sens_out=S_all[r * n_loc:(r + 1) * n_loc])
    torch.cuda.synchronize()
    seed = W.quant_seed(t)
    got = []
    for r in range(k):
        lo, hi = r * n_loc, (r + 1) * n_loc

        def gather(S_global, S_local, lo=lo, hi=hi):
            assert torch.equal(S_local, S_all[lo:hi]), "rank's own S_n"
            S_global.copy_(S_all)

        xs = [x[lo:hi].contiguous()]
        plan = ActivationSetPlan(xs, [seed], avg_bits=1.25, n_total=N, sample_base=lo,
                                 gather=gather)
        outs = [torch.empty(xs[0].numel(), dtype=torch.bfloat16, device=DEV)]
        ps = PipelinedStep(plan, outs, A.api.BF16, DEV)
        with torch.cuda.stream(ps.stream):
            ps()
        torch.cuda.synchronize()
        L = plan.layers[0]
        off = host(L.off[lo:hi + 1])
        got.append((host(L.bits[lo:hi]), host(L.packed[:int(off[-1] - off[0])]),
                    host(L.zmin).view(np.uint32), host(L.scale).view(np.uint32),
                    out_bits(outs[0], xs[0].numel())))
        del plan, ps, outs, xs
    xh = x_host(x)
    ref = O.sharded_quantize(xh, k, 1.25, seed, threads=CORES)
    D = act.D
    for r in range(k):
        bits, packed, zmin, scale, out = got[r]
        rp, rz, rs, rb = ref[r]
        assert np.array_equal(bits, rb), (r, "bits")
        assert np.array_equal(packed, rp), (r, "packed")
        assert np.array_equal(zmin, rz.ravel().view(np.uint32)), (r, "zmin")
        assert np.array_equal(scale, rs.ravel().view(np.uint32)), (r, "scale")
        exp = O.dequantize(rp, rz, rs, rb, n_loc, D, out_dtype=O.BF16, threads=CORES)
        assert np.array_equal(out, exp.ravel()), (r, "dequantised")
