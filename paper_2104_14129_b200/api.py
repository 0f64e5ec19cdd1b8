"""Python face of the ActNN hot path: thin wrappers over the C ABI.

Each function allocates its outputs as torch tensors (PyTorch is used only for
device memory and streams), passes ``data_ptr()``s and the current CUDA stream
to ``libactnn.so``, and checks the status.  No arithmetic of the method
happens here: group statistics, allocation, quantisation and dequantisation
all run in the sm_100a kernels.  Inputs must be CUDA tensors; there is no CPU
fallback.

Names follow the paper (P = PAPER.md): quantize/dequantize (§4.1),
allocate_bits (stage 1 of §4.3), group_stats (the ||R_n||^2 factor
of the sensitivity, Eq. 7-8).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import torch

from . import _lib
from ._lib import ActnnError  # noqa: F401

G = 256
F32, BF16 = 0, 1
LEVELS_POW2 = (1 << 1) | (1 << 2) | (1 << 4) | (1 << 8)
LEVELS_UNIT = 0x1FE
OP_GROUP_STATS = 0
OP_GRAD_SQNORM = 2


def library_path() -> str:
    return _lib.LIB_PATH


def abi_version() -> int:
    return int(_lib.load().actnn_abi_version())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return F32
    if dt == torch.bfloat16:
        return BF16
    raise ActnnError(-1, f"unsupported dtype {dt} (fp32 or bf16)")


def _as_2d(x: torch.Tensor) -> torch.Tensor:
    if not x.is_cuda:
        raise ActnnError(-1, "actnn needs CUDA tensors (there is no CPU fallback)")
    if not x.is_contiguous():
        raise ActnnError(-1, "actnn needs a contiguous [N, ...] activation")
    N = x.shape[0] if x.dim() > 0 else 1
    D = 1
    for s in x.shape[1:]:
        D *= s
    return x.reshape(N, D)


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def _need(t: Optional[torch.Tensor], name: str, dtype: torch.dtype, numel: Optional[int],
          device: torch.device, at_least: bool = False, optional: bool = False):
    """Validate a caller-supplied buffer before its pointer reaches the C ABI:
    a CUDA tensor on `device`, contiguous, of `dtype`, with `numel` elements
    (or at least that many).  Raises ActnnError(-1) instead of letting a wrong
    buffer turn into an out-of-bounds device access."""
    if t is None:
        if optional:
            return
        raise ActnnError(-1, f"{name} is required")
    if not t.is_cuda or t.device != device:
        raise ActnnError(-1, f"{name} must be a CUDA tensor on {device} (got {t.device})")
    if not t.is_contiguous():
        raise ActnnError(-1, f"{name} must be contiguous")
    if t.dtype != dtype:
        raise ActnnError(-1, f"{name} must be {dtype} (got {t.dtype})")
    if numel is not None:
        if (t.numel() < numel) if at_least else (t.numel() != numel):
            raise ActnnError(-1, f"{name} has {t.numel()} elements, expected "
                                 f"{'at least ' if at_least else ''}{numel}")


def packed_bytes(N: int, D: int, bits_host=None) -> int:
    """Bytes of the packed stream: sum_n b_n * ceil(D/G) * G / 8; None = 8-bit bound."""
    arr = None
    if bits_host is not None:
        import numpy as np
        arr = np.ascontiguousarray(bits_host, dtype=np.uint8)
    v = _lib.load().actnn_packed_bytes(N, D, G, None if arr is None else arr.ctypes.data_as(
        ctypes.c_void_p))
    if v < 0:
        raise ActnnError(-1, "invalid arguments to actnn_packed_bytes")
    return int(v)


@dataclass
class Packed:
    """A compressed activation (the saved context of P:578-592).

    Metadata is either fp32 (zmin, scale) or, with meta="bf16" (NEXT-1, the
    paper's P:513 format), one int32 word per group in ``meta``: bits 0-15 the
    bf16 zero point Z', bits 16-31 the bf16 range R' (zmin/scale are None)."""
    packed: torch.Tensor      # uint8 code stream, sample n at off[n] - off[0]
    zmin: Optional[torch.Tensor]   # fp32 [N * ng]  zero points Z_ni
    scale: Optional[torch.Tensor]  # fp32 [N * ng]  R_ni / B_n
    bits: torch.Tensor        # uint8 [N]      b_n
    off: torch.Tensor         # int64 [N + 1]  byte offsets
    shape: Tuple[int, ...]    # original activation shape
    dtype: torch.dtype        # original activation dtype
    seed: int
    sample_base: int
    meta: Optional[torch.Tensor] = None  # int32 [N * ng] bf16 (Z', R') words

    @property
    def N(self) -> int:
        return self.shape[0]

    @property
    def D(self) -> int:
        n = 1
        for s in self.shape[1:]:
            n *= s
        return n

    def meta_bytes(self) -> int:
        return (4 * self.meta.numel() if self.meta is not None
                else 4 * self.zmin.numel() + 4 * self.scale.numel())

    def payload_bytes(self) -> int:
        """Bytes of code stream actually used: off[N] - off[0] (one 16-byte
        device read; the widths live on the device)."""
        ends = self.off[[0, -1]].cpu()
        return int(ends[1] - ends[0])

    def nbytes(self) -> int:
        """Compressed size of the context: used code bytes + metadata + the
        per-sample widths and offsets (not the allocated capacity)."""
        return self.payload_bytes() + self.meta_bytes() + self.bits.numel() + 8 * self.off.numel()

    def capacity_bytes(self) -> int:
        """Allocated bytes (the packed buffer defaults to the 8-bit bound)."""
        return self.packed.numel() + self.meta_bytes() + self.bits.numel() + 8 * self.off.numel()


def group_stats(x: torch.Tensor, sens_out: Optional[torch.Tensor] = None):
    """Per-group canonical (min, max) and per-sample S_n = ||R_n||^2 (fp64).

    ``sens_out`` (fp64 [N], e.g. a slice of a zero-padded global vector for
    the sharded path) receives S when given."""
    x2 = _as_2d(x)
    N, D = x2.shape
    ng = ceil_div(D, G)
    dev = x2.device
    gmin = torch.empty(N * ng, dtype=torch.float32, device=dev)
    gmax = torch.empty(N * ng, dtype=torch.float32, device=dev)
    sens = sens_out if sens_out is not None else torch.empty(N, dtype=torch.float64, device=dev)
    lib = _lib.load()
    wsb = int(lib.actnn_workspace_bytes(OP_GROUP_STATS, N, D, G))
    ws = torch.zeros(max(wsb, 8), dtype=torch.uint8, device=dev)
    _lib.check(lib.actnn_group_stats(_ptr(x2), _dtype_code(x2.dtype), N, D, G, _ptr(gmin),
                                     _ptr(gmax), _ptr(sens), _ptr(ws), ws.numel(), _stream(dev)))
    return gmin, gmax, sens


def allocate_bits(sens: torch.Tensor, budget: int, D: int, level_mask: int = LEVELS_POW2,
                  gscale: Optional[torch.Tensor] = None):
    """Stage-1 greedy on the device -> (bits u8 [N], off i64 [N+1])."""
    if not sens.is_cuda:
        raise ActnnError(-1, "sens must be a CUDA fp64 tensor")
    N = sens.numel()
    dev = sens.device
    _need(sens, "sens", torch.float64, N, dev)
    _need(gscale, "gscale", torch.float64, N, dev, optional=True)
    bits = torch.empty(N, dtype=torch.uint8, device=dev)
    off = torch.empty(N + 1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().actnn_allocate_bits(_ptr(sens), _ptr(gscale), N,
                                               int(budget), level_mask, D, G, _ptr(bits),
                                               _ptr(off), None, 0, _stream(dev)))
    return bits, off


def uniform_bits(N: int, D: int, b: int, device) -> Tuple[torch.Tensor, torch.Tensor]:
    dev = torch.device(device)
    bits = torch.empty(N, dtype=torch.uint8, device=dev)
    off = torch.empty(N + 1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().actnn_uniform_bits(N, D, G, b, _ptr(bits), _ptr(off), _stream(dev)))
    return bits, off


def quantize(x: torch.Tensor, bits: torch.Tensor, off: torch.Tensor, seed: int,
             sample_base: int = 0, gmin: Optional[torch.Tensor] = None,
             gmax: Optional[torch.Tensor] = None, packed: Optional[torch.Tensor] = None,
             zmin: Optional[torch.Tensor] = None, scale: Optional[torch.Tensor] = None,
             packed_nbytes: Optional[int] = None, meta: str = "f32",
             meta_out: Optional[torch.Tensor] = None) -> Packed:
    """Compressor: per-group SR quantisation + packing.

    ``packed`` defaults to the 8-bit upper bound (bits live on the device);
    pass ``packed_nbytes`` (e.g. read back from off[N]) to size it exactly.
    ``meta="bf16"``: the paper's bf16 metadata (NEXT-1) in one int32
    word per group (``meta_out``) instead of fp32 zmin/scale."""
    x2 = _as_2d(x)
    N, D = x2.shape
    ng = ceil_div(D, G)
    dev = x2.device
    _need(bits, "bits", torch.uint8, N, dev)
    _need(off, "off", torch.int64, N + 1, dev)
    if (gmin is None) != (gmax is None):
        raise ActnnError(-1, "give both gmin and gmax (two-pass) or neither (single pass)")
    _need(gmin, "gmin", torch.float32, N * ng, dev, optional=True)
    _need(gmax, "gmax", torch.float32, N * ng, dev, optional=True)
    if packed is None:
        nbytes = packed_nbytes if packed_nbytes is not None else N * ng * G
        packed = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    else:
        # the device-resident widths decide the real size (off[N] - off[0] bytes);
        # a caller-sized buffer must hold at least packed_nbytes when given
        _need(packed, "packed", torch.uint8, packed_nbytes, dev, at_least=True)
    if meta == "bf16":
        if meta_out is None:
            meta_out = torch.empty(N * ng, dtype=torch.int32, device=dev)
        _need(meta_out, "meta_out", torch.int32, N * ng, dev)
        _lib.check(_lib.load().actnn_quantize_bf16meta(
            _ptr(x2), _dtype_code(x2.dtype), N, D, G, _ptr(bits), _ptr(off),
            ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), sample_base, _ptr(gmin), _ptr(gmax),
            _ptr(packed), _ptr(meta_out), _stream(dev)))
        return Packed(packed, None, None, bits, off, tuple(x.shape), x.dtype, seed, sample_base,
                      meta_out)
    if meta != "f32":
        raise ActnnError(-1, f"unknown metadata format {meta!r} (f32 or bf16)")
    if zmin is None:
        zmin = torch.empty(N * ng, dtype=torch.float32, device=dev)
    if scale is None:
        scale = torch.empty(N * ng, dtype=torch.float32, device=dev)
    _need(zmin, "zmin", torch.float32, N * ng, dev)
    _need(scale, "scale", torch.float32, N * ng, dev)
    _lib.check(_lib.load().actnn_quantize(
        _ptr(x2), _dtype_code(x2.dtype), N, D, G, _ptr(bits), _ptr(off),
        ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), sample_base, _ptr(gmin), _ptr(gmax),
        _ptr(packed), _ptr(zmin), _ptr(scale), _stream(dev)))
    return Packed(packed, zmin, scale, bits, off, tuple(x.shape), x.dtype, seed, sample_base)


def dequantize(p: Packed, out: Optional[torch.Tensor] = None,
               out_dtype: Optional[torch.dtype] = None) -> torch.Tensor:
    """Decompressor into a tensor of the original shape."""
    dev = p.packed.device
    N, D = p.N, p.D
    ng = ceil_div(D, G)
    if out is None:
        out = torch.empty(p.shape, dtype=out_dtype or p.dtype, device=dev)
    _need(out, "out", out.dtype if out.dtype in (torch.float32, torch.bfloat16) else torch.float32,
          N * D, dev)
    _need(p.packed, "packed", torch.uint8, None, dev)
    _need(p.bits, "bits", torch.uint8, N, dev)
    _need(p.off, "off", torch.int64, N + 1, dev)
    if p.meta is not None:
        _need(p.meta, "meta", torch.int32, N * ng, dev)
    else:
        _need(p.zmin, "zmin", torch.float32, N * ng, dev)
        _need(p.scale, "scale", torch.float32, N * ng, dev)
    if p.meta is not None:
        _lib.check(_lib.load().actnn_dequantize_bf16meta(
            _ptr(p.packed), _ptr(p.meta), _ptr(p.bits), _ptr(p.off), p.N, p.D, G, _ptr(out),
            _dtype_code(out.dtype), _stream(dev)))
        return out
    _lib.check(_lib.load().actnn_dequantize(
        _ptr(p.packed), _ptr(p.zmin), _ptr(p.scale), _ptr(p.bits), _ptr(p.off), p.N, p.D, G,
        _ptr(out), _dtype_code(out.dtype), _stream(dev)))
    return out


def compress(x: torch.Tensor, seed: int, bits: Optional[int] = None,
             avg_bits: Optional[float] = None, level_mask: int = LEVELS_POW2,
             sample_base: int = 0, gscale: Optional[torch.Tensor] = None,
             sens_allreduce: Optional[Callable[[torch.Tensor], torch.Tensor]] = None,
             n_total: Optional[int] = None, meta: str = "f32") -> Packed:
    """One layer's compress call.

    bits=b: uniform b-bit (optimization level L2, single pass).
    avg_bits=a: per-sample mixed precision (L2.5): group_stats ->
    [sens_allreduce hook: sums the zero-padded S across ranks] -> greedy
    allocation with budget floor(a * N_total) -> quantize with the stats.
    meta="bf16": the paper's bf16 per-group metadata (NEXT-1)."""
    x2 = _as_2d(x)
    N, D = x2.shape
    if bits is not None:
        b, o = uniform_bits(N, D, bits, x2.device)
        return quantize(x, b, o, seed, sample_base, meta=meta)
    if avg_bits is None:
        raise ActnnError(-1, "compress needs bits= or avg_bits=")
    nt = n_total if n_total is not None else N
    S = torch.zeros(nt, dtype=torch.float64, device=x2.device)
    gmin, gmax, _ = group_stats(x, sens_out=S[sample_base:sample_base + N] if nt != N else S)
    if sens_allreduce is not None:
        S = sens_allreduce(S)
    budget = int(avg_bits * nt)
    bits_g, off_g = allocate_bits(S, budget, D, level_mask, gscale)
    lo = sample_base if nt != N else 0
    return quantize(x, bits_g[lo:lo + N], off_g[lo:lo + N + 1], seed, sample_base, gmin, gmax,
                    meta=meta)


def decompress(p: Packed, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    return dequantize(p, out)


# --------------------------------------------------------------------- NEXT-4
# Lossless contexts (P:1388-1395 ReLU 1-bit mask; P:1406-1419 max-pool argmax).

def relu_pack(x: torch.Tensor, want_y: bool = False):
    """ReLU context: (mask u8 [ceil(E/8)], y = ReLU(x) or None), one read of x."""
    x = x.contiguous()
    if not x.is_cuda:
        raise ActnnError(-1, "relu_pack needs a CUDA tensor")
    E = x.numel()
    mask = torch.empty((E + 7) // 8, dtype=torch.uint8, device=x.device)
    y = torch.empty_like(x) if want_y else None
    _lib.check(_lib.load().actnn_relu_pack(_ptr(x), _dtype_code(x.dtype), E, _ptr(mask), _ptr(y),
                                           _stream(x.device)))
    return mask, y


def relu_backward(mask: torch.Tensor, grad_y: torch.Tensor) -> torch.Tensor:
    grad_y = grad_y.contiguous()
    if not grad_y.is_cuda:
        raise ActnnError(-1, "relu_backward needs CUDA tensors")
    _need(mask, "mask", torch.uint8, (grad_y.numel() + 7) // 8, grad_y.device)
    gx = torch.empty_like(grad_y)
    _lib.check(_lib.load().actnn_relu_backward(_ptr(mask), _ptr(grad_y),
                                               _dtype_code(grad_y.dtype), grad_y.numel(),
                                               _ptr(gx), _stream(grad_y.device)))
    return gx


def _pair(v):
    return (v, v) if isinstance(v, int) else tuple(v)


def _pool_extent(H, k, s, p, d):
    return (H + 2 * p - d * (k - 1) - 1) // s + 1


def maxpool2d(x: torch.Tensor, kernel, stride=None, padding=0, dilation=1):
    """Max pooling with its 8-bit argmax context: (y, idx u8), x [N, C, H, W]."""
    k = _pair(kernel)
    s = _pair(stride if stride is not None else kernel)
    p, d = _pair(padding), _pair(dilation)
    x = x.contiguous()
    if not x.is_cuda:
        raise ActnnError(-1, "maxpool2d needs a CUDA tensor")
    N, C, H, W = x.shape
    OH, OW = _pool_extent(H, k[0], s[0], p[0], d[0]), _pool_extent(W, k[1], s[1], p[1], d[1])
    y = torch.empty((N, C, OH, OW), dtype=x.dtype, device=x.device)
    idx = torch.empty((N, C, OH, OW), dtype=torch.uint8, device=x.device)
    _lib.check(_lib.load().actnn_maxpool2d_forward(
        _ptr(x), _dtype_code(x.dtype), N * C, H, W, k[0], k[1], s[0], s[1], p[0], p[1], d[0],
        d[1], _ptr(y), _ptr(idx), _stream(x.device)))
    return y, idx


def maxpool2d_backward(idx: torch.Tensor, grad_y: torch.Tensor, H: int, W: int, kernel,
                       stride=None, padding=0, dilation=1) -> torch.Tensor:
    k = _pair(kernel)
    s = _pair(stride if stride is not None else kernel)
    p, d = _pair(padding), _pair(dilation)
    grad_y = grad_y.contiguous()
    if not grad_y.is_cuda or grad_y.dim() != 4:
        raise ActnnError(-1, "maxpool2d_backward needs a CUDA grad_y [N, C, OH, OW]")
    N, C = grad_y.shape[:2]
    OH, OW = _pool_extent(H, k[0], s[0], p[0], d[0]), _pool_extent(W, k[1], s[1], p[1], d[1])
    if tuple(grad_y.shape[2:]) != (OH, OW):
        raise ActnnError(-1, f"grad_y is {tuple(grad_y.shape)}, the pooling geometry gives "
                             f"[{N}, {C}, {OH}, {OW}]")
    _need(idx, "idx", torch.uint8, grad_y.numel(), grad_y.device)
    gx = torch.empty((N, C, H, W), dtype=grad_y.dtype, device=grad_y.device)
    _lib.check(_lib.load().actnn_maxpool2d_backward(
        _ptr(idx), _ptr(grad_y), _dtype_code(grad_y.dtype), N * C, H, W, k[0], k[1], s[0], s[1],
        p[0], p[1], d[0], d[1], _ptr(gx), _stream(grad_y.device)))
    return gx


# --------------------------------------------------------------------- NEXT-3
# Run-time adaptation: gradient-magnitude factor, its estimators,
# stage-2 per-layer allocation.

def grad_sqnorm(grad: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Per-sample ||grad_n||^2 (fp64 [N]) of a gradient tensor [N, ...]."""
    g2 = _as_2d(grad)
    N, D = g2.shape
    dev = g2.device
    out = out if out is not None else torch.empty(N, dtype=torch.float64, device=dev)
    lib = _lib.load()
    wsb = int(lib.actnn_workspace_bytes(OP_GRAD_SQNORM, N, D, G))
    ws = torch.zeros(max(wsb, 8), dtype=torch.uint8, device=dev)
    _lib.check(lib.actnn_grad_sqnorm(_ptr(g2), _dtype_code(g2.dtype), N, D, G, _ptr(out),
                                     _ptr(ws), ws.numel(), _stream(dev)))
    return out


def gradmag_ema(obs: torch.Tensor, m: torch.Tensor, rho: float = 0.9) -> torch.Tensor:
    """Moving average across samples: m (fp64 [1], device) updated in place."""
    if obs.dtype != torch.float64 or m.dtype != torch.float64 or not obs.is_cuda:
        raise ActnnError(-1, "gradmag_ema needs CUDA fp64 tensors")
    obs = obs.contiguous()
    _lib.check(_lib.load().actnn_gradmag_ema(_ptr(obs), obs.numel(), float(rho), _ptr(m),
                                             _stream(obs.device)))
    return m


def gradmag_gather(table: torch.Tensor, ids: torch.Tensor) -> torch.Tensor:
    """Stale estimator: est[n] = table[ids[n]]."""
    ids = ids.contiguous()
    if not table.is_cuda:
        raise ActnnError(-1, "gradmag_gather needs CUDA tensors")
    _need(table, "table", torch.float64, None, table.device)
    _need(ids, "ids", torch.int64, None, table.device)
    est = torch.empty(ids.numel(), dtype=torch.float64, device=table.device)
    _lib.check(_lib.load().actnn_gradmag_gather(_ptr(table), table.numel(), _ptr(ids),
                                                ids.numel(), _ptr(est), _stream(table.device)))
    return est


def gradmag_scatter(table: torch.Tensor, ids: torch.Tensor, obs: torch.Tensor) -> torch.Tensor:
    """Stale estimator update: table[ids[n]] = obs[n] (in place)."""
    ids, obs = ids.contiguous(), obs.contiguous()
    if not table.is_cuda:
        raise ActnnError(-1, "gradmag_scatter needs CUDA tensors")
    _need(table, "table", torch.float64, None, table.device)
    _need(ids, "ids", torch.int64, None, table.device)
    _need(obs, "obs", torch.float64, ids.numel(), table.device)
    _lib.check(_lib.load().actnn_gradmag_scatter(_ptr(table), table.numel(), _ptr(ids),
                                                 _ptr(obs), ids.numel(), _stream(table.device)))
    return table


class LayerAllocator:
    """Stage 2 with a persistent zero-initialised workspace for L
    layers of N samples: ``__call__(sens [L, N], b_total)`` -> (bits [L, N] u8,
    budgets [L] i64), on the device in one cooperative launch."""

    def __init__(self, D, N: int, device, level_mask: int = LEVELS_POW2):
        self.D = [int(d) for d in D]
        self.L, self.N = len(self.D), int(N)
        self.level_mask = level_mask
        self.dev = torch.device(device)
        lib = _lib.load()
        wsb = int(lib.actnn_allocate_layers_ws_bytes(self.L, self.N, level_mask))
        self.ws = torch.zeros(max(wsb, 256), dtype=torch.uint8, device=self.dev)
        self._D_host = (ctypes.c_int64 * max(self.L, 1))(*self.D)

    def __call__(self, sens: torch.Tensor, b_total: int, gscale: Optional[torch.Tensor] = None,
                 lconst: Optional[torch.Tensor] = None):
        if sens.dtype != torch.float64 or not sens.is_cuda:
            raise ActnnError(-1, "sens must be a CUDA fp64 tensor [L, N]")
        sens = sens.contiguous()
        gscale = gscale.contiguous() if gscale is not None else None
        lconst = lconst.contiguous() if lconst is not None else None
        _need(sens, "sens", torch.float64, self.L * self.N, self.dev)
        _need(gscale, "gscale", torch.float64, self.L * self.N, self.dev, optional=True)
        _need(lconst, "lconst", torch.float64, self.L, self.dev, optional=True)
        bits = torch.empty((self.L, self.N), dtype=torch.uint8, device=self.dev)
        budgets = torch.empty(self.L, dtype=torch.int64, device=self.dev)
        _lib.check(_lib.load().actnn_allocate_layers(
            _ptr(sens), _ptr(gscale), _ptr(lconst), self._D_host, self.L, self.N, int(b_total),
            self.level_mask, _ptr(bits), _ptr(budgets), _ptr(self.ws), self.ws.numel(),
            _stream(self.dev)))
        return bits, budgets


def allocate_layers(sens: torch.Tensor, D, b_total: int, level_mask: int = LEVELS_POW2,
                    gscale: Optional[torch.Tensor] = None, lconst: Optional[torch.Tensor] = None):
    """One-shot stage-2 allocation (a fresh workspace per call)."""
    L, N = sens.shape
    return LayerAllocator(D, N, sens.device, level_mask)(sens, b_total, gscale, lconst)
