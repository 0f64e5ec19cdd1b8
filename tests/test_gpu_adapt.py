"""GPU vs oracle parity of the NEXT-3 run-time adaptation kernels
through the C ABI: per-sample gradient norms (O14), the moving-average and
stale estimators (O15-O16) and the stage-2 joint allocation (O17).  fp64
outputs and widths are compared bit for bit (the kernels follow the oracle's
summation and key order exactly)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2104_14129_b200 as A
    return A


def to_oracle(t):
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def f64_bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


# ------------------------------------------------------------------ O14
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("N,D", [(1, 256), (3, 1000), (4, 256 * 70), (5, 256 * 33 + 17),
                                 (7, 3 * 224 * 224), (2, 64 * 56 * 56), (64, 2048), (3, 5)])
def test_grad_sqnorm_parity(A, dtype, N, D):
    g = torch.Generator(device=DEV).manual_seed(N * 1000 + D)
    x = (torch.randn((N, D), generator=g, device=DEV)
         * torch.exp(torch.randn((N, 1), generator=g, device=DEV) * 3)).to(dtype)
    x[:, ::11] = 0.0
    out = A.grad_sqnorm(x)
    ref = O.grad_sqnorm(to_oracle(x))
    assert np.array_equal(f64_bits(out.cpu().numpy()), f64_bits(ref))
    # misaligned view -> the generic (non-vector) kernel, same bits
    buf = torch.empty(N * D + 1, dtype=dtype, device=DEV)
    xv = buf[1:].view(N, D)
    xv.copy_(x)
    assert np.array_equal(f64_bits(A.grad_sqnorm(xv).cpu().numpy()), f64_bits(ref))


def test_grad_sqnorm_edges(A):
    out = A.grad_sqnorm(torch.empty((4, 0), device=DEV))
    assert out.cpu().tolist() == [0.0] * 4
    assert A.grad_sqnorm(torch.empty((0, 256), device=DEV)).numel() == 0
    x = torch.zeros((2, 512), device=DEV)
    x[0, 511] = 2.0 ** 40
    x[1, 0] = -(2.0 ** -60)
    assert A.grad_sqnorm(x).cpu().tolist() == [2.0 ** 80, 2.0 ** -120]
    # the workspace ticket is left at zero: repeated calls agree
    y = torch.randn((33, 4096), device=DEV)
    a, b = A.grad_sqnorm(y), A.grad_sqnorm(y)
    assert torch.equal(a, b)


# ------------------------------------------------------------------ O15 / O16
@pytest.mark.parametrize("N", [1, 31, 32, 33, 1000, 4096])
def test_gradmag_ema_parity(A, N):
    rng = np.random.default_rng(N)
    m_dev = torch.ones(1, dtype=torch.float64, device=DEV)
    m_ref = 1.0
    for step in range(5):
        obs = 10 ** rng.uniform(-3, 3, N)
        A.gradmag_ema(torch.from_numpy(obs).to(DEV), m_dev, 0.9)
        m_ref = O.gradmag_ema(obs, m_ref, 0.9)
    assert f64_bits([m_dev.item()])[0] == f64_bits([m_ref])[0]


def test_gradmag_stale_table(A):
    T = 10000
    table = torch.ones(T, dtype=torch.float64, device=DEV)
    rng = np.random.default_rng(0)
    ids = rng.permutation(T)[:1024]
    obs = rng.random(1024)
    ids_d = torch.from_numpy(ids).to(DEV)
    assert A.gradmag_gather(table, ids_d).cpu().tolist() == [1.0] * 1024
    A.gradmag_scatter(table, ids_d, torch.from_numpy(obs).to(DEV))
    ref = O.gradmag_scatter(np.ones(T), ids, obs)
    assert np.array_equal(table.cpu().numpy(), ref)
    ids2 = rng.integers(0, T, 777)
    est = A.gradmag_gather(table, torch.from_numpy(ids2).to(DEV)).cpu().numpy()
    assert np.array_equal(est, O.gradmag_gather(ref, ids2))


# ------------------------------------------------------------------ O17
def _stage2(A, sens, D, tot, mask, gscale=None, lconst=None, alloc=None):
    L, N = sens.shape
    s_d = torch.from_numpy(np.ascontiguousarray(sens)).to(DEV)
    g_d = None if gscale is None else torch.from_numpy(np.ascontiguousarray(gscale)).to(DEV)
    c_d = None if lconst is None else torch.from_numpy(np.ascontiguousarray(lconst)).to(DEV)
    alloc = alloc or A.LayerAllocator(D, N, DEV, mask)
    bits, bud = alloc(s_d, tot, g_d, c_d)
    rb, rbud = O.allocate_layers(sens, D, tot, mask, gscale, lconst)
    assert np.array_equal(bits.cpu().numpy(), rb)
    assert np.array_equal(bud.cpu().numpy(), rbud)
    return rb, rbud


def _resnet_dims(name):
    return [a.D for a in W.workload(name).acts]


@pytest.mark.parametrize("mask", [O.LEVELS_POW2, O.LEVELS_UNIT])
@pytest.mark.parametrize("avg", [1.25, 2.0, 3.3])
def test_stage2_resnet50_parity(A, mask, avg):
    """ResNet-50 layer dims, N = 256, S_n drawn like the C3 workload (per-sample
    lognormal scale, per-layer decades), total budget avg bits/element."""
    D = _resnet_dims("c3")
    L, N = len(D), 256
    rng = np.random.default_rng(int(avg * 100) + mask)
    sens = (np.exp(2 * rng.standard_normal((1, N))) * 10 ** rng.uniform(-3, 3, (L, 1))
            * np.asarray(D, np.float64)[:, None])
    tot = int(avg * N * sum(D))
    _stage2(A, sens, D, tot, mask)


def test_stage2_resnet152_c4_size(A):
    """C4's stage-2 problem: 311 layers x 1024 samples (955k moves), 1.25 bits,
    with per-sample gradient estimates and per-layer constants."""
    D = _resnet_dims("c4")
    L, N = len(D), 1024
    rng = np.random.default_rng(152)
    sens = np.exp(rng.standard_normal((L, N))) * 10 ** rng.uniform(-2, 2, (L, 1))
    gscale = np.exp(rng.standard_normal((L, N)))
    lconst = rng.uniform(0.01, 10, L)
    _stage2(A, sens, D, int(1.25 * N * sum(D)), O.LEVELS_POW2, gscale, lconst)


def test_stage2_ties_and_edges(A):
    rng = np.random.default_rng(7)
    D = [3, 256, 17, 256, 1000, 5]
    L, N = len(D), 64
    full = 8 * N * sum(D)
    floor = N * sum(D)
    alloc = A.LayerAllocator(D, N, DEV, O.LEVELS_POW2)
    # all-equal sensitivities: huge key ties, the index-order cut (> 32 moves share a key)
    for tot in (floor, floor + 1, 2 * floor + 7, 5 * floor - 3, full - 1, full, full + 100):
        _stage2(A, np.ones((L, N)), D, tot, O.LEVELS_POW2, alloc=alloc)
    # zero sensitivities (key 0) mixed with positives; a dominant sample
    s = 10 ** rng.uniform(-3, 3, (L, N))
    s[rng.random((L, N)) < 0.4] = 0.0
    s[2, 5] = 1e12
    for tot in (floor, 2 * floor, 3 * floor + 11):
        _stage2(A, s, D, tot, O.LEVELS_POW2, alloc=alloc)
        _stage2(A, s, D, tot, O.LEVELS_UNIT)
    # one layer == the stage-1 allocator (same ABI family, D = 1)
    s1 = 10 ** rng.uniform(-3, 3, (1, 300))
    b2, _ = _stage2(A, s1, [1], 600, O.LEVELS_POW2)
    b1, _ = A.allocate_bits(torch.from_numpy(s1[0]).to(DEV), 600, 256)
    assert np.array_equal(b1.cpu().numpy(), b2[0])
    # infeasible budget raises, N = 0 gives zero budgets
    with pytest.raises(A.ActnnError):
        A.allocate_layers(torch.ones((2, 3), dtype=torch.float64, device=DEV), [4, 4], 23)
    z = A.LayerAllocator([4, 4], 0, DEV)(torch.empty((2, 0), dtype=torch.float64, device=DEV), 0)
    assert z[1].cpu().tolist() == [0, 0]
