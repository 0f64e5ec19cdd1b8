"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test states the passage (P:<line> = PAPER.md, S:<line> = SPEC.md) or the
mathematical fact it checks.  None of them re-types the oracle's formulas: they
use known-answer vectors, worked examples produced by an independent
transcription, closed forms, exhaustive enumeration, brute force, Monte Carlo
against the paper's mean/variance law, and invariants.
"""
import hashlib
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------- Philox
def test_philox_known_answer_vectors():
    """Random123 KAT (tests/golden/philox_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        out = O.philox4x32_10(v[0:4], v[4:6])
        assert list(out) == v[6:10]
        n += 1
    assert n == 3


def test_random14_uniform_chi_square():
    """The 14-bit draws feeding stochastic rounding are uniform (needed for
    E[u_hat] = u_bar): chi-square over 64 bins on 2^16 elements."""
    r = np.array([O.random14(12345, e) for e in range(1 << 16)])
    assert r.min() >= 0 and r.max() < (1 << 14)
    counts = np.bincount(r >> 8, minlength=64)
    exp = len(r) / 64
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    assert chi2 < 120.0  # df = 63; p(chi2 > 120) < 1e-5


# --------------------------------------------------------------------------- worked examples
def _worked():
    return json.load(open(os.path.join(GOLD, "worked_examples.json")))


def test_worked_example_W1():
    w = _worked()["W1"]
    x = (np.arange(256, dtype=np.float32) / np.float32(255)).reshape(1, 256)
    assert [f"{v:08x}" for v in O.philox4x32_10([0, 0, 0, 0], [42, 0])] == w["philox_ctr0_key42"]
    packed, zmin, scale, off = O.quantize(x, w["bits"], w["seed"], w["sample_base"])
    assert zmin.ravel().tolist() == w["zmin"]
    assert [f"{v:08x}" for v in scale.view(np.uint32).ravel()] == w["scale_bits_hex"]
    assert len(packed) == w["packed_len"] and off[-1] == w["packed_len"]
    assert packed[:16].tobytes().hex() == w["packed_prefix_hex"]
    assert hashlib.sha256(packed.tobytes()).hexdigest()[:16] == w["packed_sha256_prefix"]
    codes, _ = O.dequantize_group(packed, 256, 2, zmin[0, 0], scale[0, 0])
    assert codes[:16].tolist() == w["codes_sample0_first16"]


def test_worked_example_W2():
    w = _worked()["W2"]
    d = np.arange(1024)
    x = ((((37 * d) % 101) - 50).astype(np.float32) / np.float32(8)).reshape(2, 512)
    packed, zmin, scale, off = O.quantize(x, np.array(w["bits"], np.uint8), w["seed"],
                                          w["sample_base"])
    assert zmin.ravel().tolist() == w["zmin"]
    assert np.allclose(scale.ravel(), w["scale"], rtol=0, atol=1e-9)
    assert len(packed) == w["packed_len"]
    assert hashlib.sha256(packed.tobytes()).hexdigest()[:16] == w["packed_sha256_prefix"]
    c0, _ = O.dequantize_group(packed[off[0]:], 8, 1, zmin[0, 0], scale[0, 0])
    c1, _ = O.dequantize_group(packed[off[1]:], 8, 8, zmin[1, 0], scale[1, 0])
    assert c0.tolist() == w["codes_sample0_first8"]
    assert c1.tolist() == w["codes_sample1_first8"]


# --------------------------------------------------------------------------- quantiser
@pytest.mark.parametrize("b", [1, 2, 4, 8])
@pytest.mark.parametrize("e", [-3, 0, 5])
def test_grid_values_round_trip_exactly(b, e):
    """Values on the quantisation grid Z + k*R/B are reproduced exactly and
    deterministically: the rounding has nothing to round."""
    rng = np.random.default_rng(b * 10 + e)
    B = (1 << b) - 1
    k = rng.integers(0, B + 1, size=256)
    k[3], k[200] = 0, B                       # the group spans the whole grid
    step = np.float32(2.0 ** e)
    Z = np.float32(-37.0) * step
    h = (Z + k.astype(np.float32) * step).astype(np.float32)
    for seed in (0, 1, 99):
        seg, z, s = O.quantize_group(h, b, seed, 1000 + seed)
        codes, out = O.dequantize_group(seg, 256, b, z, s)
        assert codes.tolist() == k.tolist()
        assert np.array_equal(out, h)


def test_spec_examples_grid_and_constant():
    """S:129/S:138 [0,1,2,3] at 2 bits -> codes [0,1,2,3]; S:130/S:139 constant
    group [5,5,5,5] -> codes 0, Z = 5, exact."""
    seg, z, s = O.quantize_group(np.array([0, 1, 2, 3], np.float32), 2, 7, 0)
    codes, out = O.dequantize_group(seg, 4, 2, z, s)
    assert codes.tolist() == [0, 1, 2, 3] and out.tolist() == [0, 1, 2, 3]
    assert seg[0] == 0xE4  # 0b11_10_01_00 under the LSB-first layout
    seg, z, s = O.quantize_group(np.full(4, 5.0, np.float32), 4, 7, 0)
    codes, out = O.dequantize_group(seg, 4, 4, z, s)
    assert z == 5.0 and codes.tolist() == [0] * 4 and out.tolist() == [5.0] * 4


def test_packing_layout_spec_examples():
    """codes [1,2,3] at 2 bits are the byte 0x39; [1] at 1 bit is 0x01.
    Packing (via grid values [0,3,2,1] -> 0x6C) and unpacking both checked."""
    codes, _ = O.dequantize_group(np.array([0x39, 0], np.uint8), 3, 2, 0.0, 1.0)
    assert codes.tolist() == [1, 2, 3]
    codes, _ = O.dequantize_group(np.array([0x01], np.uint8), 1, 1, 0.0, 1.0)
    assert codes.tolist() == [1]
    seg, _, _ = O.quantize_group(np.array([0, 3, 2, 1], np.float32), 2, 1, 0)
    assert seg[0] == 0x6C and seg[1:].sum() == 0     # padding codes are 0
    seg, _, _ = O.quantize_group(np.array([0, 1, 0, 0, 0, 0, 0, 0, 1], np.float32), 1, 1, 0)
    assert seg[0] == 0x02 and seg[1] == 0x01


@pytest.mark.parametrize("b", [1, 2, 4, 8])
def test_code_range_and_extremes(b):
    """0 <= code <= B; min maps to 0 and max to B deterministically."""
    rng = np.random.default_rng(b)
    B = (1 << b) - 1
    for trial in range(20):
        h = (rng.standard_normal(256) * 10 ** rng.uniform(-3, 3) + rng.uniform(-50, 50))
        h = h.astype(np.float32)
        seg, z, s = O.quantize_group(h, b, trial, trial * 256)
        codes, _ = O.dequantize_group(seg, 256, b, z, s)
        assert codes.max() <= B
        assert codes[np.argmin(h)] == 0 and codes[np.argmax(h)] == B
        assert z == h.min()


def test_stochastic_rounding_probability():
    """u_hat = ceil(u_bar) with probability u_bar - floor(u_bar).
    Group [0, 1, 0.25 x 254] at b=1: Z=0, R=1, u_bar = 0.25 for 254 elements,
    so P(code = 1) = 0.25 exactly; 200 seeds x 254 draws, 5-sigma band."""
    h = np.full(256, 0.25, np.float32)
    h[0], h[1] = 0.0, 1.0
    ones = 0
    for seed in range(200):
        seg, z, s = O.quantize_group(h, 1, seed, seed * 4096)
        codes, _ = O.dequantize_group(seg, 256, 1, z, s)
        ones += int(codes[2:].sum())
    n = 200 * 254
    p = ones / n
    assert abs(p - 0.25) < 5 * math.sqrt(0.25 * 0.75 / n)


@pytest.mark.parametrize("b", [1, 2, 4])
def test_unbiased_and_variance_law_per_element(b):
    """Thm 1 needs E[h_hat] = h; the per-element variance of stochastic
    rounding is p(1-p) scale^2 with p = frac(u_bar) (north_star).
    Monte Carlo over 4000 seeds, 4-SE band on the mean plus the fixed-point
    resolution 2^-14 scale (DESIGN reading 6)."""
    rng = np.random.default_rng(100 + b)
    h = (rng.standard_normal(256) * 2 + 3).astype(np.float32)
    S = 4000
    acc = np.zeros(256)
    acc2 = np.zeros(256)
    for seed in range(S):
        seg, z, s = O.quantize_group(h, b, seed, 7 * 256)
        _, out = O.dequantize_group(seg, 256, b, z, s)
        acc += out
        acc2 += out.astype(np.float64) ** 2
    mean = acc / S
    var = acc2 / S - mean ** 2
    B = (1 << b) - 1
    R = float(h.max()) - float(h.min())
    scale = R / B
    u = (h.astype(np.float64) - float(h.min())) / scale
    p = u - np.floor(u)
    vth = p * (1 - p) * scale ** 2
    se = np.sqrt(np.maximum(vth, 1e-30) / S)
    assert np.all(np.abs(mean - h) <= 4 * se + scale * 2.0 ** -14 + 1e-6 * abs(h).max())
    # variance: aggregate over the 256 elements (relative SE ~ 1/sqrt(S*256))
    assert abs(var.sum() / vth.sum() - 1.0) < 0.05


def test_variance_law_uniform_data():
    """P:512 / S:158: for U(0,1) fractional parts, Var = R^2/(6 B^2) per element
    (~0.0185 at R ~ 1, B = 3), within 10%; 4 -> 2 bits multiplies it by 25."""
    rng = np.random.default_rng(5)
    h = rng.random(256).astype(np.float32)
    def emp_var(b, S=600):
        acc = np.zeros(256); acc2 = np.zeros(256)
        for seed in range(S):
            seg, z, s = O.quantize_group(h, b, seed, 0)
            _, out = O.dequantize_group(seg, 256, b, z, s)
            acc += out; acc2 += out.astype(np.float64) ** 2
        return float(np.mean(acc2 / S - (acc / S) ** 2))
    R = float(h.max() - h.min())
    v2 = emp_var(2)
    assert abs(v2 / (R * R / (6 * 9)) - 1) < 0.10
    v4 = emp_var(4)
    assert abs((v2 / v4) / 25.0 - 1) < 0.2


def test_degenerate_and_tiny_ranges():
    """R = 0 -> all codes 0 and h_hat = Z; R < 2^-96 is treated
    the same (DESIGN reading 16) while scale keeps RN(R/B)."""
    h = np.full(256, 1.0, np.float32)
    h[9] = np.float32(1.0) + np.float32(2.0 ** -23)
    seg, z, s = O.quantize_group(h, 2, 3, 0)
    codes, _ = O.dequantize_group(seg, 256, 2, z, s)
    assert set(codes[h == 1.0].tolist()) == {0} and z == 1.0
    tiny = np.zeros(256, np.float32)
    tiny[4] = np.float32(2.0 ** -100)
    seg, z, s = O.quantize_group(tiny, 8, 3, 0)
    codes, out = O.dequantize_group(seg, 256, 8, z, s)
    assert codes.max() == 0 and z == 0.0 and s == np.float32(2.0 ** -100) / np.float32(255)


def test_nondegenerate_tiny_ranges():
    """Tiny but non-degenerate ranges (R in {2^-100, 2^-90};
    DESIGN reading 16 puts the threshold at 2^-96), where inv14 = RN(B/R) 2^14
    reaches ~B 2^110 and members may be subnormal.
    (1) Grid round trip: values k 2^-97, R = 3 2^-97 > 2^-96, b = 2 ->
        codes = k and h_hat = h exactly.
    (2) The threshold itself: R = 2^-96 quantises (non-zero codes), the float
        just below it is degenerate (all codes 0, h_hat = Z).
    (3) Unbiasedness for a group spanning [0, 2^-95] with subnormal
        and zero members: Monte Carlo mean within 4 SE + 2^-14 scale."""
    k = np.arange(256) % 4
    h = (k * np.float32(2.0 ** -97)).astype(np.float32)
    h[0], h[1] = 0.0, np.float32(3 * 2.0 ** -97)
    seg, z, s = O.quantize_group(h, 2, 11, 0)
    codes, out = O.dequantize_group(seg, 256, 2, z, s)
    k[0], k[1] = 0, 3
    assert np.array_equal(codes, k) and np.array_equal(out, h)

    rng = np.random.default_rng(5)
    for R, degenerate in ((np.float32(2.0 ** -96), False),
                          (np.nextafter(np.float32(2.0 ** -96), np.float32(0)), True)):
        g = (rng.random(256) * float(R)).astype(np.float32)
        g[0], g[1] = 0.0, R
        seg, z, s = O.quantize_group(g, 4, 3, 0)
        codes, out = O.dequantize_group(seg, 256, 4, z, s)
        if degenerate:
            assert codes.max() == 0 and np.all(out == 0.0)
        else:
            assert codes.max() == 15 and np.count_nonzero(codes) > 200
            assert np.all(np.abs(out.astype(np.float64) - g) <= float(s))

    g = (rng.random(256) * 2.0 ** -95).astype(np.float32)
    g[2::3] = (rng.random(85) * 2.0 ** -126).astype(np.float32)   # subnormal members
    g[4::7] = 0.0
    g[0], g[1] = 0.0, np.float32(2.0 ** -95)
    assert np.count_nonzero((g > 0) & (g < 2.0 ** -126)) > 50
    b, S = 2, 3000
    acc = np.zeros(256)
    for seed in range(S):
        seg, z, s = O.quantize_group(g, b, seed, 3 * 256)
        _, out = O.dequantize_group(seg, 256, b, z, s)
        acc += out.astype(np.float64)
    scale = float(s)
    u = g.astype(np.float64) / scale
    p = u - np.floor(u)
    se = np.sqrt(np.maximum(p * (1 - p), 1e-30) / S) * scale
    assert np.all(np.abs(acc / S - g) <= 4 * se + scale * 2.0 ** -14)


def test_signed_zero_canonical():
    """DESIGN reading 17: Z is canonical +0 whether the group's zeros are +0 or -0."""
    h = np.zeros(256, np.float32)
    h[1::2] = -0.0
    _, z, s = O.quantize_group(h, 2, 0, 0)
    assert np.signbit(z) == False and np.signbit(s) == False  # noqa: E712
    _, z, _ = O.quantize_group(-np.zeros(256, np.float32), 2, 0, 0)
    assert np.signbit(z) == False  # noqa: E712


def test_bf16_input_and_output():
    """bf16 input widens exactly (same codes as the fp32 copy); bf16 output is
    RNE of the fp32 value (checked against torch's RNE cast, a library routine)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    xf = rng.standard_normal((3, 512)).astype(np.float32)
    xb = torch.from_numpy(xf).to(torch.bfloat16)
    xb_bits = xb.view(torch.int16).numpy().view(np.uint16)
    xw = xb.float().numpy()
    bits = np.array([1, 4, 8], np.uint8)
    p1 = O.quantize(xb_bits, bits, 5, 0)
    p2 = O.quantize(xw, bits, 5, 0)
    for a, b in zip(p1, p2):
        assert np.array_equal(a, b)
    packed, zmin, scale, _ = p2
    out32 = O.dequantize(packed, zmin, scale, bits, 3, 512)
    out16 = O.dequantize(packed, zmin, scale, bits, 3, 512, out_dtype=O.BF16)
    ref = torch.from_numpy(out32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(out16, ref)


def test_ragged_groups_and_threads():
    """Ragged last group: only real elements enter Z/R, padding
    codes are 0; results do not depend on the thread count."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 700)).astype(np.float32)   # ng = 3, last group 188
    bits = np.array([1, 2, 4, 8, 2], np.uint8)
    a = O.quantize(x, bits, 9, 2, threads=1)
    b = O.quantize(x, bits, 9, 2, threads=3)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    packed, zmin, scale, off = a
    assert off[-1] == 3 * 32 * int(bits.sum())
    for n in range(5):
        assert zmin[n, 2] == x[n, 512:].min()
        b = int(bits[n])
        seg = packed[off[n] + 2 * 32 * b: off[n] + 3 * 32 * b]
        codes, _ = O.dequantize_group(seg, 256, b, zmin[n, 2], scale[n, 2])
        assert codes[188:].max() == 0
    out = O.dequantize(packed, zmin, scale, bits, 5, 700)
    step = scale.repeat(256, axis=1)[:, :700].astype(np.float64)
    assert np.all(np.abs(out - x) <= step * (1 + 1e-6))   # |h_hat - h| <= one step R/B


def test_sharding_invariance():
    """O13: k virtual ranks (slices with sample_base, global allocation over the
    summed zero-padded S) reproduce the 1-rank bytes exactly."""
    rng = np.random.default_rng(21)
    x = (rng.standard_normal((8, 512)) * np.exp(rng.standard_normal((8, 1)))).astype(np.float32)
    one = O.sharded_quantize(x, 1, 2.0, 77)[0]
    for k in (2, 4, 8):
        parts = O.sharded_quantize(x, k, 2.0, 77)
        cat = [np.concatenate([p[i] for p in parts]) for i in range(4)]
        for u, v in zip(cat, one):
            assert np.array_equal(u, v)


# --------------------------------------------------------------------------- stats
def test_group_ranges_spec_examples():
    """[0,1,2,3] -> R = 3, ||R||^2 = 9; groups [0,2],[1,5] -> R = [2,4],
    ||R||^2 = 20; constant tensor -> ranges 0."""
    gmin, gmax = O.group_minmax(np.array([[0, 1, 2, 3]], np.float32), G=4)
    assert (gmax - gmin).tolist() == [[3.0]] and O.sensitivity(gmin, gmax).tolist() == [9.0]
    gmin, gmax = O.group_minmax(np.array([[0, 2, 1, 5]], np.float32), G=2)
    assert (gmax - gmin).tolist() == [[2.0, 4.0]]
    assert O.sensitivity(gmin, gmax).tolist() == [20.0]
    gmin, gmax = O.group_minmax(np.full((2, 600), 3.5, np.float32), G=256)
    assert (gmax - gmin).max() == 0 and O.sensitivity(gmin, gmax).max() == 0


def test_sensitivity_matches_exact_sum():
    """S_n equals the exactly rounded sum of R_ni^2 (math.fsum) to within the
    error bound of a 5 + nch term fp64 summation; ranges equal the brute-force
    max - min."""
    rng = np.random.default_rng(8)
    x = (rng.standard_normal((6, 256 * 70)) * rng.uniform(0.01, 100, (6, 1))).astype(np.float32)
    gmin, gmax = O.group_minmax(x, 256)
    g = x.reshape(6, 70, 256)
    assert np.array_equal(gmin, g.min(axis=2)) and np.array_equal(gmax, g.max(axis=2))
    S = O.sensitivity(gmin, gmax)
    for n in range(6):
        R = (gmax[n] - gmin[n]).astype(np.float64)
        exact = math.fsum(R * R)
        assert abs(S[n] - exact) <= 16 * 2.0 ** -53 * exact


# --------------------------------------------------------------------------- allocator
def test_allocator_spec_examples():
    """S:329, S:338-340, S:355-356 examples and feasibility errors."""
    assert O.objective(np.array([4.0, 1.0]), np.array([2, 2], np.uint8)) == pytest.approx(5 / 9)
    for mask in (O.LEVELS_POW2, O.LEVELS_UNIT):
        bits = O.allocate_bits(np.array([16.0, 1.0]), 6, mask)
        assert bits.tolist() == [4, 2]
        assert O.objective(np.array([16.0, 1.0]), bits) == pytest.approx(16 / 225 + 1 / 9)
        assert O.allocate_bits(np.array([1e6, 1.0]), 9, mask).tolist() == [8, 1]
        w = np.random.default_rng(0).random(10)
        assert O.allocate_bits(w, 80, mask).tolist() == [8] * 10
        assert O.allocate_bits(w, 10, mask).tolist() == [1] * 10
        assert O.allocate_bits(np.ones(7), 14, mask).tolist() == [2] * 7
        with pytest.raises(ValueError):
            O.allocate_bits(w, 9, mask)
    # zero-sensitivity samples sink first
    assert O.allocate_bits(np.array([0.0, 1.0, 0.0]), 10, O.LEVELS_POW2).tolist() == [1, 8, 1]


def test_dp_equals_bruteforce():
    """The knapsack DP and exhaustive search agree on tiny instances."""
    rng = np.random.default_rng(1)
    for mask in (O.LEVELS_POW2, O.LEVELS_UNIT):
        for _ in range(150):
            N = int(rng.integers(1, 5))
            w = 10 ** rng.uniform(-3, 3, N)
            budget = int(rng.integers(N, 8 * N + 1))
            ob, _ = O.allocate_bruteforce(w, budget, mask)
            od, bd = O.allocate_dp(w, budget, mask)
            assert od == pytest.approx(ob, rel=1e-12)
            assert int(bd.sum()) <= budget


def test_unit_step_greedy_is_optimal():
    """With unit steps 8,7,...,1 the greedy on a separable convex objective is
    exact (Gross 1956 / Fox 1966): greedy == brute force == DP."""
    rng = np.random.default_rng(2)
    for _ in range(400):
        N = int(rng.integers(1, 6))
        w = 10 ** rng.uniform(-3, 3, N)
        budget = int(rng.integers(N, 8 * N + 1))
        g = O.allocate_bits(w, budget, O.LEVELS_UNIT)
        ob, _ = O.allocate_bruteforce(w, budget, O.LEVELS_UNIT)
        assert int(g.sum()) <= budget
        assert O.objective(w, g) == pytest.approx(ob, rel=1e-12, abs=1e-300)
    w = 10 ** rng.uniform(-3, 3, 40)
    g = O.allocate_bits(w, 100, O.LEVELS_UNIT)
    od, _ = O.allocate_dp(w, 100, O.LEVELS_UNIT)
    assert O.objective(w, g) == pytest.approx(od, rel=1e-12)


def _last_move_increase(w, bits):
    """Absolute variance increase of the last greedy move, recomputed from the
    output bits (priority = increase per freed bit; DESIGN reading 9)."""
    L = [8, 4, 2, 1]
    f = {b: 1.0 / ((2 ** b - 1) ** 2) for b in L}
    best = None
    for n, b in enumerate(bits):
        for j in range(L.index(int(b))):
            inc = w[n] * (f[L[j + 1]] - f[L[j]])
            key = (inc / (L[j] - L[j + 1]), n, j)
            if best is None or key > best[0]:
                best = (key, inc)
    return 0.0 if best is None else best[1]


def test_level_set_greedy_bound():
    """Hot-path level set {8,4,2,1}: OPT <= greedy <= OPT + (increase of the
    last move), equality when the final total hits the budget exactly."""
    rng = np.random.default_rng(4)
    for _ in range(400):
        N = int(rng.integers(1, 6))
        w = 10 ** rng.uniform(-3, 3, N)
        budget = int(rng.integers(N, 8 * N + 1))
        g = O.allocate_bits(w, budget, O.LEVELS_POW2)
        ob, _ = O.allocate_bruteforce(w, budget, O.LEVELS_POW2)
        og = O.objective(w, g)
        assert int(g.sum()) <= budget
        assert og >= ob * (1 - 1e-12)
        assert og <= ob + _last_move_increase(w, g) * (1 + 1e-9) + 1e-300


def test_allocator_monotone_and_scale_invariant():
    """more budget never raises the objective; scaling every w by a
    power of two leaves the bits unchanged."""
    rng = np.random.default_rng(6)
    for mask in (O.LEVELS_POW2, O.LEVELS_UNIT):
        w = 10 ** rng.uniform(-4, 4, 64)
        prev = None
        for budget in range(64, 8 * 64 + 1, 7):
            obj = O.objective(w, O.allocate_bits(w, budget, mask))
            if prev is not None:
                assert obj <= prev * (1 + 1e-12)
            prev = obj
        for budget in (64, 100, 128, 333):
            assert np.array_equal(O.allocate_bits(w, budget, mask),
                                  O.allocate_bits(w * 1024.0, budget, mask))


def test_allocator_mixed_beats_uniform():
    """S:390 (mixed-precision dominance): at an equal budget 2N the greedy's
    Eq. 8 objective is <= the uniform 2-bit objective."""
    rng = np.random.default_rng(7)
    for _ in range(50):
        w = np.exp(2 * rng.standard_normal(32))
        g = O.allocate_bits(w, 64, O.LEVELS_POW2)
        assert O.objective(w, g) <= O.objective(w, np.full(32, 2, np.uint8)) * (1 + 1e-12)


def test_offsets_and_storage_accounting():
    """Payload bytes = sum_n b_n * ceil(D/G) * G / 8; fp32 metadata
    is 8 bytes per group = 0.25 bits/elem at G = 256 (DESIGN reading 4: the
    paper's bf16 pair is 0.125 bits)."""
    bits = np.array([1, 2, 4, 8], np.uint8)
    off = O.offsets(bits, 1000, 256)
    assert off.tolist() == [0, 128, 384, 896, 1920]
    assert 8 * 8 / 256 == 0.25 and 32 / 256 == 0.125
