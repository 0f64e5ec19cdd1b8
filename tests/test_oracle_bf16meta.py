"""Pins of the oracle's NEXT-1 mode: bf16 per-group metadata ("store the
per-group range and zero points in bfloat16, so each group costs extra 32
bits, which is 0.125 bits on average"; "rounded to bfloat16
BEFORE scaling (stored and used values identical)"; DESIGN reading 21).

The reading: Z' = the largest bf16 <= Z, R' = the smallest bf16 >= M - Z'
(exact), so [Z', Z' + R'] contains the group and E[h_hat] = h still holds.
The pins below check that definition against an enumeration of every finite
bf16 value with exact rational arithmetic, and the statistical and closed-form
properties the paper states, on the tensor-level quantize/dequantize.
"""
import bisect
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

# every finite bf16 value, exactly, ascending (a bf16 is an fp32 with zero low half)
_pat = (np.arange(1 << 16, dtype=np.uint32) << np.uint32(16)).view(np.float32)
_BF16 = np.unique(_pat[np.isfinite(_pat)].astype(np.float64))  # -0 and +0 merge
_BF16_FR = [Fraction(float(v)) for v in _BF16]


def _floor_bf16(z: float) -> float:
    """Largest bf16 <= z (z an fp32 value, exact in float64)."""
    i = int(np.searchsorted(_BF16, z, side="right")) - 1
    return float(_BF16[i])


def _ceil_bf16_exact(x: Fraction) -> float:
    """Smallest bf16 >= x, x an exact rational."""
    i = bisect.bisect_left(_BF16_FR, x)
    return float(_BF16[i])


def _fields(w: int):
    Z, R = O.meta_fields(np.array([w], np.uint32))
    return float(Z[0]), float(R[0])


def _cases():
    rng = np.random.default_rng(2104)
    out = []
    for _ in range(3000):
        a = rng.standard_normal() * 10.0 ** rng.uniform(-30, 30)
        b = a + abs(rng.standard_normal()) * 10.0 ** rng.uniform(-30, 30)
        out.append((np.float32(a), np.float32(max(a, b))))
    special = [0.0, 1.0, -1.0, 5.0, 0.1, -0.1, 1e-40, -1e-40, 2.0 ** -126, 3.0, 2.0 ** 100,
               -2.0 ** 100, 1.0 + 2.0 ** -8, 1.0 + 2.0 ** -9, -(1.0 + 2.0 ** -9), 255.0]
    for z in special:
        for m in special:
            if m >= z:
                out.append((np.float32(z), np.float32(m)))
    return out


def test_meta_is_the_tightest_outward_bf16_pair():
    """Z' = max{bf16 <= Z} and R' = min{bf16 >= M - Z'} by enumeration of all
    65536 bf16 patterns with exact rational arithmetic; hence
    Z' <= Z <= M <= Z' + R' (containment)."""
    for Z, M in _cases():
        Z = np.float32(Z + np.float32(0.0))  # canonical +0 as O3
        Zp, Rp = _fields(O.meta_bf16(Z, M))
        assert Zp == _floor_bf16(float(Z)), (Z, M)
        exact = Fraction(float(M)) - Fraction(Zp)
        assert Rp == _ceil_bf16_exact(exact), (Z, M)
        assert Fraction(Zp) <= Fraction(float(Z))
        assert Fraction(Zp) + Fraction(Rp) >= Fraction(float(M))


def test_spec_grid_and_constant_examples_with_bf16_meta():
    """[0,1,2,3] at b=2 -> codes 0..3 and exact
    round trip (0 and 3 are bf16 values); [5,5,5,5] -> R' = 0, codes 0, 5."""
    x = np.array([[0, 1, 2, 3] + [3] * 252], np.float32)
    packed, meta, off = O.quantize_bf16meta(x, 2, seed=9)
    assert _fields(int(meta[0, 0])) == (0.0, 3.0)
    out = O.dequantize_bf16meta(packed, meta, [2], 1, 256)
    assert np.array_equal(out, x)
    c = np.full((1, 256), 5.0, np.float32)
    packed, meta, off = O.quantize_bf16meta(c, 4, seed=1)
    assert _fields(int(meta[0, 0])) == (5.0, 0.0)
    assert not packed.any()
    assert np.array_equal(O.dequantize_bf16meta(packed, meta, [4], 1, 256), c)


def test_grid_round_trip_on_bf16_exact_metadata():
    """Values Z + k R/B with bf16-exact Z, R and R/B a power of two: codes are
    deterministic and h_hat == h exactly."""
    for b in (1, 2, 4, 8):
        B = (1 << b) - 1
        step = 2.0 ** -3
        Z = -1.5
        k = np.arange(256) % (B + 1)
        k[0], k[1] = 0, B
        x = (Z + k * step).astype(np.float32).reshape(1, 256)
        packed, meta, _ = O.quantize_bf16meta(x, b, seed=b)
        Zp, Rp = _fields(int(meta[0, 0]))
        assert (Zp, Rp) == (Z, B * step)
        assert np.array_equal(O.dequantize_bf16meta(packed, meta, [b], 1, 256), x)


@pytest.mark.parametrize("b", [1, 2, 4])
def test_unbiased_with_bf16_meta(b):
    """P:510 E[h_hat] = h must survive the metadata rounding (DESIGN reading
    21: the quantiser uses the stored, outward-rounded values).  Group with a
    non-bf16 minimum (so Z' < Z strictly); Monte Carlo over 1500 seeds, 4-SE
    band plus the 2^-14 fixed-point resolution."""
    rng = np.random.default_rng(40 + b)
    h = (0.1 + rng.random(256) * 0.7).astype(np.float32).reshape(1, 256)
    S = 1500
    acc = np.zeros(256)
    acc2 = np.zeros(256)
    for seed in range(S):
        packed, meta, _ = O.quantize_bf16meta(h, b, seed=seed)
        out = O.dequantize_bf16meta(packed, meta, [b], 1, 256)[0].astype(np.float64)
        acc += out
        acc2 += out ** 2
    Zp, Rp = _fields(int(meta[0, 0]))
    assert Zp < float(h.min()) and Zp + Rp >= float(h.max())
    scale = Rp / ((1 << b) - 1)
    mean = acc / S
    # SE from the SR variance law p(1-p) scale^2, p = frac(u_bar)
    u = (h[0].astype(np.float64) - Zp) / scale
    pf = u - np.floor(u)
    se = np.sqrt(pf * (1 - pf) / S) * scale
    assert np.all(np.abs(mean - h[0]) <= 4 * se + scale * 2.0 ** -14 + 1e-7)
    emp = acc2 / S - mean ** 2
    assert abs(emp.sum() / (pf * (1 - pf) * scale ** 2).sum() - 1.0) < 0.06


def test_constant_non_bf16_group_is_unbiased():
    """A constant group at 0.1 (not a bf16 value): Z' < 0.1 < Z' + R', so the
    codes are stochastic and the mean of h_hat is 0.1."""
    x = np.full((1, 256), 0.1, np.float32)
    S = 400
    acc = 0.0
    ones = 0
    for seed in range(S):
        packed, meta, _ = O.quantize_bf16meta(x, 1, seed=seed)
        ones += int(np.unpackbits(packed).sum())
        acc += float(O.dequantize_bf16meta(packed, meta, [1], 1, 256).astype(np.float64).mean())
    Zp, Rp = _fields(int(meta[0, 0]))
    p = (0.1 - Zp) / Rp
    n = S * 256
    assert abs(ones / n - p) < 5 * math.sqrt(p * (1 - p) / n)
    assert abs(acc / S - float(np.float32(0.1))) < 5 * Rp * math.sqrt(p * (1 - p) / n) + 1e-7


def test_code_range_and_invariant_on_wide_inputs():
    """0 <= code <= B and the q <= B 2^14 invariant hold
    with outward-rounded metadata on ranges from 2^-90 to 2^100 and mixed
    signs (the oracle raises if the invariant fails)."""
    rng = np.random.default_rng(77)
    rows = []
    for e in (-90, -20, 0, 20, 100):
        rows.append(rng.standard_normal(256) * 2.0 ** e)
        rows.append(-np.abs(rng.standard_normal(256)) * 2.0 ** e - 3 * 2.0 ** e)
    x = np.asarray(rows, np.float32)
    for b in (1, 2, 3, 4, 8):
        packed, meta, off = O.quantize_bf16meta(x, b, seed=b)
        out = O.dequantize_bf16meta(packed, meta, [b] * len(x), len(x), 256)
        Z, R = O.meta_fields(meta)
        lo = Z.astype(np.float64)
        hi = lo + R.astype(np.float64)
        slack = np.abs(hi) * 2.0 ** -23 + 1e-45
        assert np.all(out >= lo[:, :1] - slack[:, :1]) and np.all(out <= hi[:, :1] + slack[:, :1])


def test_variance_law_with_bf16_meta():
    """P:512 / S:158 with the stored range: uniform [0,1) data, b = 2 ->
    per-element variance ~ R'^2/(6 B^2) (~0.0185) within 10%."""
    rng = np.random.default_rng(5)
    x = rng.random(256).astype(np.float32).reshape(1, 256)
    S = 500
    acc = np.zeros(256)
    acc2 = np.zeros(256)
    for seed in range(S):
        packed, meta, _ = O.quantize_bf16meta(x, 2, seed=seed)
        out = O.dequantize_bf16meta(packed, meta, [2], 1, 256)[0].astype(np.float64)
        acc += out
        acc2 += out ** 2
    _, Rp = _fields(int(meta[0, 0]))
    v = float(np.mean(acc2 / S - (acc / S) ** 2))
    assert abs(v / (Rp * Rp / 54.0) - 1) < 0.10


def test_memory_arithmetic_of_the_paper():
    """32 bits per group = 0.125 bits/element at G = 256; P:826-828:
    a Conv-BN-ReLU block at 2 bits costs 2.125 + 2.125 + 1 = 5.25 bits versus
    64, i.e. ~12x.  Counted from the oracle's buffers."""
    N, D, b = 4, 1024, 2
    x = np.random.default_rng(0).random((N, D)).astype(np.float32)
    packed, meta, off = O.quantize_bf16meta(x, b, seed=3)
    bits_per_elem = 8 * (packed.nbytes + meta.nbytes) / (N * D)
    assert bits_per_elem == b + 0.125
    block = 2 * bits_per_elem + 1.0  # conv + bn inputs, 1-bit ReLU mask (NEXT-4)
    assert block == 5.25 and round(64 / block) == 12


def test_tensor_level_matches_groups_threads_and_bf16_io():
    """The tensor routines equal the per-group routine (ragged last group,
    sample_base offset, thread count), and bf16 output is torch's RNE cast of
    the fp32 output (a library routine)."""
    import torch
    rng = np.random.default_rng(8)
    N, D, G = 3, 700, 256
    x = (rng.standard_normal((N, D)) * 3).astype(np.float32)
    bits = [1, 4, 8]
    packed, meta, off = O.quantize_bf16meta(x, bits, seed=11, sample_base=5, threads=3)
    ng = 3
    for n in range(N):
        for i in range(ng):
            h = x[n, i * G:min((i + 1) * G, D)]
            seg, w = O.quantize_group_bf16meta(h, bits[n], 11, (5 + n) * D + i * G)
            s0 = off[n] + i * G * bits[n] // 8
            assert np.array_equal(packed[s0:s0 + len(seg)], seg)
            assert int(meta[n, i]) == w
    f32 = O.dequantize_bf16meta(packed, meta, bits, N, D)
    b16 = O.dequantize_bf16meta(packed, meta, bits, N, D, out_dtype=O.BF16, threads=2)
    ref = torch.from_numpy(f32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(b16, ref)
