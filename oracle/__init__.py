"""CPU oracle for the ActNN hot path ("ACTNN-Q v1"), ctypes binding.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2104_14129_b200`` never imports it and
shares no code with it ("Oracle").

Every function is a thin numpy marshalling layer over ``actnn_oracle.cpp``;
the arithmetic lives there, each step citing the PAPER.md passage it follows.
Functions without an external pin would say "parity unpinned" here; none do
(the pins are listed in DESIGN.md, "Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

F32, BF16 = 0, 1
LEVELS_POW2 = (1 << 1) | (1 << 2) | (1 << 4) | (1 << 8)   # {1,2,4,8}, the hot path
LEVELS_UNIT = 0x1FE                                      # 1..8, the paper's unit step
ERR_BUDGET = -3


def build() -> str:
    """Compile liboracle.so with the oracle's own Makefile (-ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        src = os.path.join(_HERE, "actnn_oracle.cpp")
        if (not os.path.exists(_LIB_PATH)
                or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        P, I64, I32, U64, U32 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                 ctypes.c_uint64, ctypes.c_uint32)
        sig = {
            "oracle_philox4x32_10": (None, [P, P, P]),
            "oracle_random14": (U32, [U64, U64]),
            "oracle_group_minmax": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P, P]),
            "oracle_sensitivity": (None, [P, P, I64, I64, P]),
            "oracle_allocate_bits": (ctypes.c_int, [P, I64, I64, U32, P]),
            "oracle_objective": (ctypes.c_double, [P, P, I64]),
            "oracle_allocate_bruteforce": (ctypes.c_double, [P, I64, I64, U32, P]),
            "oracle_allocate_dp": (ctypes.c_double, [P, I64, I64, U32, P]),
            "oracle_offsets": (None, [P, I64, I64, I32, P]),
            "oracle_quantize_group": (ctypes.c_int, [P, I32, I32, I32, U64, U64, P, P, P]),
            "oracle_quantize": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P, U64, I64,
                                               P, P, P, ctypes.c_int]),
            "oracle_dequantize": (ctypes.c_int, [P, P, P, P, I64, I64, I32, P, ctypes.c_int,
                                                 ctypes.c_int]),
            "oracle_dequantize_group": (None, [P, I32, I32, ctypes.c_float, ctypes.c_float,
                                               P, P]),
            "oracle_meta_bf16": (U32, [ctypes.c_float, ctypes.c_float]),
            "oracle_quantize_group_bf16meta": (ctypes.c_int, [P, I32, I32, I32, U64, U64, P, P]),
            "oracle_quantize_bf16meta": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P, U64,
                                                        I64, P, P, ctypes.c_int]),
            "oracle_dequantize_bf16meta": (ctypes.c_int, [P, P, P, I64, I64, I32, P,
                                                          ctypes.c_int, ctypes.c_int]),
            "oracle_relu_pack": (ctypes.c_int, [P, ctypes.c_int, I64, P, P]),
            "oracle_relu_backward": (ctypes.c_int, [P, P, ctypes.c_int, I64, P]),
            "oracle_maxpool2d_forward": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I64] + [I32] * 8
                                         + [I64, I64, P, P]),
            "oracle_maxpool2d_backward": (ctypes.c_int, [P, P, ctypes.c_int, I64, I64, I64]
                                          + [I32] * 8 + [I64, I64, P]),
            "oracle_grad_sqnorm": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P]),
            "oracle_gradmag_ema": (ctypes.c_int, [P, I64, ctypes.c_double, P]),
            "oracle_gradmag_gather": (ctypes.c_int, [P, I64, P, I64, P]),
            "oracle_gradmag_scatter": (ctypes.c_int, [P, I64, P, P, I64]),
            "oracle_allocate_layers": (ctypes.c_int, [P, P, P, P, I64, I64, I64, U32, P, P]),
            "oracle_objective_layers": (ctypes.c_double, [P, P, P, I64, I64, P]),
            "oracle_allocate_layers_dp": (ctypes.c_double, [P, P, P, P, I64, I64, I64, U32, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _as_x(x: np.ndarray):
    """fp32 arrays pass as F32; bf16 tensors pass as their uint16 bit patterns."""
    x = np.ascontiguousarray(x)
    if x.dtype == np.float32:
        return x, F32
    if x.dtype == np.uint16:
        return x, BF16
    raise TypeError(f"oracle input must be float32 or uint16 (bf16 bits), got {x.dtype}")


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    _load().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o


def random14(seed: int, e: int) -> int:
    return int(_load().oracle_random14(seed, e))


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def group_minmax(x: np.ndarray, G: int = 256):
    """x: [N, D] fp32 or bf16 bits -> (gmin, gmax) each [N, ceil(D/G)] fp32."""
    x, dt = _as_x(x)
    N, D = x.shape
    ng = ceil_div(D, G)
    gmin = np.zeros((N, ng), np.float32)
    gmax = np.zeros((N, ng), np.float32)
    st = _load().oracle_group_minmax(_ptr(x), dt, N, D, G, _ptr(gmin), _ptr(gmax))
    assert st == 0, st
    return gmin, gmax


def sensitivity(gmin: np.ndarray, gmax: np.ndarray) -> np.ndarray:
    """S_n = ||R_n||^2 in the canonical order (fp64 [N])."""
    gmin = np.ascontiguousarray(gmin, np.float32)
    gmax = np.ascontiguousarray(gmax, np.float32)
    N, ng = gmin.shape
    S = np.zeros(N, np.float64)
    _load().oracle_sensitivity(_ptr(gmin), _ptr(gmax), N, ng, _ptr(S))
    return S


def allocate_bits(w: np.ndarray, budget: int, level_mask: int = LEVELS_POW2) -> np.ndarray:
    """Heap greedy.  Raises ValueError when the budget is infeasible."""
    w = np.ascontiguousarray(w, np.float64)
    bits = np.zeros(len(w), np.uint8)
    st = _load().oracle_allocate_bits(_ptr(w), len(w), int(budget), level_mask, _ptr(bits))
    if st != 0:
        raise ValueError(f"oracle_allocate_bits failed: {st}")
    return bits


def objective(w: np.ndarray, bits: np.ndarray) -> float:
    w = np.ascontiguousarray(w, np.float64)
    bits = np.ascontiguousarray(bits, np.uint8)
    return float(_load().oracle_objective(_ptr(w), _ptr(bits), len(w)))


def allocate_bruteforce(w, budget, level_mask=LEVELS_POW2):
    w = np.ascontiguousarray(w, np.float64)
    bits = np.zeros(len(w), np.uint8)
    obj = _load().oracle_allocate_bruteforce(_ptr(w), len(w), int(budget), level_mask,
                                             _ptr(bits))
    return obj, bits


def allocate_dp(w, budget, level_mask=LEVELS_POW2):
    w = np.ascontiguousarray(w, np.float64)
    bits = np.zeros(len(w), np.uint8)
    obj = _load().oracle_allocate_dp(_ptr(w), len(w), int(budget), level_mask, _ptr(bits))
    return obj, bits


def offsets(bits: np.ndarray, D: int, G: int = 256) -> np.ndarray:
    bits = np.ascontiguousarray(bits, np.uint8)
    off = np.zeros(len(bits) + 1, np.int64)
    _load().oracle_offsets(_ptr(bits), len(bits), D, G, _ptr(off))
    return off


def quantize_group(h: np.ndarray, b: int, seed: int, e0: int, G: int = 256):
    """One group (len(h) <= G) whose first element has global index e0.
    Returns (segment bytes [G*b/8], zmin, scale)."""
    h = np.ascontiguousarray(h, np.float32)
    seg = np.zeros(G * b // 8, np.uint8)
    z = ctypes.c_float()
    s = ctypes.c_float()
    st = _load().oracle_quantize_group(_ptr(h), len(h), G, b, seed, e0, _ptr(seg),
                                       ctypes.byref(z), ctypes.byref(s))
    if st != 0:
        raise ValueError(f"oracle_quantize_group failed: {st}")
    return seg, np.float32(z.value), np.float32(s.value)


def quantize(x: np.ndarray, bits, seed: int, sample_base: int = 0, G: int = 256,
             threads: int = 1):
    """x [N, D] -> (packed u8 [off[N]], zmin [N, ng], scale [N, ng], off [N+1])."""
    x, dt = _as_x(x)
    N, D = x.shape
    bits = np.ascontiguousarray(np.broadcast_to(np.asarray(bits, np.uint8), (N,)))
    off = offsets(bits, D, G)
    ng = ceil_div(D, G)
    packed = np.zeros(int(off[-1]), np.uint8)
    zmin = np.zeros((N, ng), np.float32)
    scale = np.zeros((N, ng), np.float32)
    st = _load().oracle_quantize(_ptr(x), dt, N, D, G, _ptr(bits), seed, sample_base,
                                 _ptr(packed), _ptr(zmin), _ptr(scale), threads)
    if st != 0:
        raise ValueError(f"oracle_quantize failed: {st}")
    return packed, zmin, scale, off


def dequantize(packed, zmin, scale, bits, N: int, D: int, G: int = 256,
               out_dtype: int = F32, threads: int = 1) -> np.ndarray:
    """-> [N, D] fp32, or uint16 bf16 bit patterns when out_dtype == BF16."""
    bits = np.ascontiguousarray(np.broadcast_to(np.asarray(bits, np.uint8), (N,)))
    packed = np.ascontiguousarray(packed, np.uint8)
    zmin = np.ascontiguousarray(zmin, np.float32)
    scale = np.ascontiguousarray(scale, np.float32)
    out = np.zeros((N, D), np.float32 if out_dtype == F32 else np.uint16)
    st = _load().oracle_dequantize(_ptr(packed), _ptr(zmin), _ptr(scale), _ptr(bits), N, D, G,
                                   _ptr(out), out_dtype, threads)
    if st != 0:
        raise ValueError(f"oracle_dequantize failed: {st}")
    return out


def dequantize_group(seg, length: int, b: int, zmin: float, scale: float):
    seg = np.ascontiguousarray(seg, np.uint8)
    codes = np.zeros(length, np.uint32)
    out = np.zeros(length, np.float32)
    _load().oracle_dequantize_group(_ptr(seg), length, b, float(zmin), float(scale),
                                    _ptr(codes), _ptr(out))
    return codes, out


# ---------------------------------------------------------------- NEXT-1
# bf16 metadata (DESIGN reading 21): one uint32 word
# per group, low half = Z' (bf16 toward -inf of Z), high half = R' (bf16
# toward +inf of RU32(M - Z')); quantisation and dequantisation use float(Z'),
# float(R').

def meta_bf16(Z: float, M: float) -> int:
    """The group's metadata word from its canonical min Z and max M."""
    return int(_load().oracle_meta_bf16(float(np.float32(Z)), float(np.float32(M))))


def meta_fields(meta) -> tuple:
    """Split words into (Z', R') as float32 arrays (exact widening)."""
    w = np.ascontiguousarray(meta, np.uint32)
    Z = (w << np.uint32(16)).view(np.float32)
    R = (w & np.uint32(0xFFFF0000)).view(np.float32)
    return Z, R


def quantize_group_bf16meta(h: np.ndarray, b: int, seed: int, e0: int, G: int = 256):
    """One group -> (segment bytes [G*b/8], metadata word)."""
    h = np.ascontiguousarray(h, np.float32)
    seg = np.zeros(G * b // 8, np.uint8)
    m = ctypes.c_uint32()
    st = _load().oracle_quantize_group_bf16meta(_ptr(h), len(h), G, b, seed, e0, _ptr(seg),
                                                ctypes.byref(m))
    if st != 0:
        raise ValueError(f"oracle_quantize_group_bf16meta failed: {st}")
    return seg, int(m.value)


def quantize_bf16meta(x: np.ndarray, bits, seed: int, sample_base: int = 0, G: int = 256,
                      threads: int = 1):
    """x [N, D] -> (packed u8 [off[N]], meta u32 [N, ng], off [N+1])."""
    x, dt = _as_x(x)
    N, D = x.shape
    bits = np.ascontiguousarray(np.broadcast_to(np.asarray(bits, np.uint8), (N,)))
    off = offsets(bits, D, G)
    ng = ceil_div(D, G)
    packed = np.zeros(int(off[-1]), np.uint8)
    meta = np.zeros((N, ng), np.uint32)
    st = _load().oracle_quantize_bf16meta(_ptr(x), dt, N, D, G, _ptr(bits), seed, sample_base,
                                          _ptr(packed), _ptr(meta), threads)
    if st != 0:
        raise ValueError(f"oracle_quantize_bf16meta failed: {st}")
    return packed, meta, off


def dequantize_bf16meta(packed, meta, bits, N: int, D: int, G: int = 256,
                        out_dtype: int = F32, threads: int = 1) -> np.ndarray:
    bits = np.ascontiguousarray(np.broadcast_to(np.asarray(bits, np.uint8), (N,)))
    packed = np.ascontiguousarray(packed, np.uint8)
    meta = np.ascontiguousarray(meta, np.uint32)
    out = np.zeros((N, D), np.float32 if out_dtype == F32 else np.uint16)
    st = _load().oracle_dequantize_bf16meta(_ptr(packed), _ptr(meta), _ptr(bits), N, D, G,
                                            _ptr(out), out_dtype, threads)
    if st != 0:
        raise ValueError(f"oracle_dequantize_bf16meta failed: {st}")
    return out


# ---------------------------------------------------------------- NEXT-4
# Lossless contexts (P:1388-1395 ReLU, P:1406-1419 max pooling).

def _dt_of(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.uint16:
        return BF16
    raise TypeError(a.dtype)


def relu_pack(x: np.ndarray, want_y: bool = False):
    """x (any shape, fp32 or bf16 bits) -> (mask u8 [ceil(E/8)], y or None)."""
    x = np.ascontiguousarray(x)
    E = x.size
    mask = np.zeros((E + 7) // 8, np.uint8)
    y = np.zeros_like(x) if want_y else None
    st = _load().oracle_relu_pack(_ptr(x), _dt_of(x), E, _ptr(mask),
                                  _ptr(y) if y is not None else None)
    assert st == 0, st
    return mask, y


def relu_backward(mask: np.ndarray, gy: np.ndarray) -> np.ndarray:
    gy = np.ascontiguousarray(gy)
    mask = np.ascontiguousarray(mask, np.uint8)
    gx = np.zeros_like(gy)
    st = _load().oracle_relu_backward(_ptr(mask), _ptr(gy), _dt_of(gy), gy.size, _ptr(gx))
    assert st == 0, st
    return gx


def pool_out(H, k, s, p, d):
    return (H + 2 * p - d * (k - 1) - 1) // s + 1


def maxpool2d_forward(x: np.ndarray, k, s, p=(0, 0), d=(1, 1)):
    """x [N, C, H, W] -> (y [N, C, OH, OW], idx u8 [N, C, OH, OW])."""
    x = np.ascontiguousarray(x)
    N, C, H, W = x.shape
    OH, OW = pool_out(H, k[0], s[0], p[0], d[0]), pool_out(W, k[1], s[1], p[1], d[1])
    y = np.zeros((N, C, OH, OW), x.dtype)
    idx = np.zeros((N, C, OH, OW), np.uint8)
    st = _load().oracle_maxpool2d_forward(_ptr(x), _dt_of(x), N * C, H, W, k[0], k[1], s[0],
                                          s[1], p[0], p[1], d[0], d[1], OH, OW, _ptr(y),
                                          _ptr(idx))
    if st != 0:
        raise ValueError(f"oracle_maxpool2d_forward failed: {st}")
    return y, idx


def maxpool2d_backward(idx: np.ndarray, gy: np.ndarray, H: int, W: int, k, s, p=(0, 0),
                       d=(1, 1)) -> np.ndarray:
    gy = np.ascontiguousarray(gy)
    idx = np.ascontiguousarray(idx, np.uint8)
    N, C, OH, OW = gy.shape
    gx = np.zeros((N, C, H, W), gy.dtype)
    st = _load().oracle_maxpool2d_backward(_ptr(idx), _ptr(gy), _dt_of(gy), N * C, H, W, k[0],
                                           k[1], s[0], s[1], p[0], p[1], d[0], d[1], OH, OW,
                                           _ptr(gx))
    if st != 0:
        raise ValueError(f"oracle_maxpool2d_backward failed: {st}")
    return gx


def sharded_quantize(x: np.ndarray, k: int, avg_bits: float, seed: int,
                     level_mask: int = LEVELS_POW2, G: int = 256, threads: int = 1):
    """O13: k virtual ranks.  Rank r owns samples [r*N/k, (r+1)*N/k); it writes
    its S_n into a zero array of length N, the k arrays are summed (the
    all-reduce), every rank allocates over all N samples with budget
    floor(avg_bits * N), then quantizes its slice with sample_base = r*N/k.
    Returns the per-rank (packed, zmin, scale, bits) tuples."""
    x, _ = _as_x(x)
    N, D = x.shape
    assert N % k == 0
    n_loc = N // k
    total = np.zeros(N, np.float64)
    for r in range(k):
        gmin, gmax = group_minmax(x[r * n_loc:(r + 1) * n_loc], G)
        part = np.zeros(N, np.float64)
        part[r * n_loc:(r + 1) * n_loc] = sensitivity(gmin, gmax)
        total = total + part
    bits = allocate_bits(total, int(np.floor(avg_bits * N)), level_mask)
    out = []
    for r in range(k):
        sl = slice(r * n_loc, (r + 1) * n_loc)
        packed, zmin, scale, _ = quantize(x[sl], bits[sl], seed, r * n_loc, G, threads)
        out.append((packed, zmin, scale, bits[sl]))
    return out


# ---------------------------------------------------------------- NEXT-3
def grad_sqnorm(g: np.ndarray, G: int = 256) -> np.ndarray:
    """O14: per-sample ||grad_n||^2 (fp64 [N]) of g [N, D] (fp32 or bf16 bits)."""
    g, dt = _as_x(g)
    N, D = g.shape
    out = np.zeros(N, np.float64)
    st = _load().oracle_grad_sqnorm(_ptr(g), dt, N, D, G, _ptr(out))
    assert st == 0, st
    return out


def gradmag_ema(obs: np.ndarray, m: float, rho: float = 0.9) -> float:
    """O15: one moving-average update m <- rho m + (1 - rho) mean(obs)."""
    obs = np.ascontiguousarray(obs, np.float64)
    mm = np.array([m], np.float64)
    st = _load().oracle_gradmag_ema(_ptr(obs), len(obs), float(rho), _ptr(mm))
    if st != 0:
        raise ValueError(f"oracle_gradmag_ema failed: {st}")
    return float(mm[0])


def gradmag_gather(table: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """O16: est[n] = table[ids[n]] (the stale estimate from the last epoch)."""
    table = np.ascontiguousarray(table, np.float64)
    ids = np.ascontiguousarray(ids, np.int64)
    est = np.zeros(len(ids), np.float64)
    st = _load().oracle_gradmag_gather(_ptr(table), len(table), _ptr(ids), len(ids), _ptr(est))
    if st != 0:
        raise ValueError(f"oracle_gradmag_gather failed: {st}")
    return est


def gradmag_scatter(table: np.ndarray, ids: np.ndarray, obs: np.ndarray) -> np.ndarray:
    """O16: table[ids[n]] = obs[n]; returns the updated copy."""
    table = np.array(table, np.float64)
    ids = np.ascontiguousarray(ids, np.int64)
    obs = np.ascontiguousarray(obs, np.float64)
    st = _load().oracle_gradmag_scatter(_ptr(table), len(table), _ptr(ids), _ptr(obs), len(ids))
    if st != 0:
        raise ValueError(f"oracle_gradmag_scatter failed: {st}")
    return table


def _opt(a, dtype=np.float64):
    if a is None:
        return None, None
    a = np.ascontiguousarray(a, dtype)
    return a, _ptr(a)


def allocate_layers(sens, D, b_total: int, level_mask: int = LEVELS_POW2, gscale=None,
                    lconst=None):
    """O17: stage-2 joint greedy.  sens/gscale [L, N], lconst [L], D [L]
    -> (bits [L, N] u8, budgets [L] i64).  Raises ValueError when infeasible."""
    sens = np.ascontiguousarray(sens, np.float64)
    L, N = sens.shape
    Da = np.ascontiguousarray(D, np.int64)
    gs, gsp = _opt(gscale)
    lc, lcp = _opt(lconst)
    bits = np.zeros((L, N), np.uint8)
    budgets = np.zeros(L, np.int64)
    st = _load().oracle_allocate_layers(_ptr(sens), gsp, lcp, _ptr(Da), L, N, int(b_total),
                                        level_mask, _ptr(bits), _ptr(budgets))
    if st != 0:
        raise ValueError(f"oracle_allocate_layers failed: {st}")
    return bits, budgets


def objective_layers(sens, bits, gscale=None, lconst=None) -> float:
    sens = np.ascontiguousarray(sens, np.float64)
    L, N = sens.shape
    bits = np.ascontiguousarray(bits, np.uint8)
    gs, gsp = _opt(gscale)
    lc, lcp = _opt(lconst)
    return float(_load().oracle_objective_layers(_ptr(sens), gsp, lcp, L, N, _ptr(bits)))


def allocate_layers_dp(sens, D, b_total: int, level_mask: int = LEVELS_POW2, gscale=None,
                       lconst=None):
    """Exact knapsack DP of Eq. 8 over all layers (tiny instances)."""
    sens = np.ascontiguousarray(sens, np.float64)
    L, N = sens.shape
    Da = np.ascontiguousarray(D, np.int64)
    gs, gsp = _opt(gscale)
    lc, lcp = _opt(lconst)
    bits = np.zeros((L, N), np.uint8)
    obj = _load().oracle_allocate_layers_dp(_ptr(sens), gsp, lcp, _ptr(Da), L, N, int(b_total),
                                            level_mask, _ptr(bits))
    return obj, bits
