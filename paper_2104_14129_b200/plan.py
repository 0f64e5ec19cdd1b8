"""Preallocated per-step executor for a whole activation set.

A training step compresses every saved activation of the network in the
forward pass and decompresses it in the backward pass (Fig. 2).
``ActivationSetPlan`` owns all per-layer buffers, prebuilds the ctypes
argument tuples of every C-ABI call, and issues the calls on the current
stream with no per-call allocation, so the CPU stays ahead of the GPU even for
the small layers.  Mixed precision (L2.5) runs per layer
  actnn_group_stats -> [all-gather of S over the ranks, k > 1]
  -> actnn_allocate_bits -> actnn_quantize (with the stats);
uniform precision (L2) runs actnn_quantize single-pass with fixed widths.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import torch

from . import _lib
from .api import BF16, F32, G, LEVELS_POW2, OP_GROUP_STATS, ceil_div

_P = ctypes.c_void_p


def _p(t: torch.Tensor, offset_elems: int = 0) -> ctypes.c_void_p:
    return _P(t.data_ptr() + offset_elems * t.element_size())


@dataclass
class Layer:
    x: torch.Tensor
    N: int
    D: int
    ng: int
    dt: int
    seed: int
    budget: int
    gmin: torch.Tensor = None
    gmax: torch.Tensor = None
    S: torch.Tensor = None          # fp64 [N_total] (global vector)
    S_loc: torch.Tensor = None      # fp64 [N] this rank's slice (a view of S when k = 1)
    ws: torch.Tensor = None
    bits: torch.Tensor = None       # u8 [N_total]
    off: torch.Tensor = None        # i64 [N_total + 1]
    packed: torch.Tensor = None
    zmin: torch.Tensor = None
    scale: torch.Tensor = None
    meta: torch.Tensor = None       # int32 [N * ng] bf16 (Z', R') words (meta="bf16")
    args: dict = field(default_factory=dict)


class ActivationSetPlan:
    def __init__(self, xs: Sequence[torch.Tensor], seeds: Sequence[int],
                 avg_bits: Optional[float] = None, bits: Optional[int] = None,
                 level_mask: int = LEVELS_POW2, n_total: Optional[int] = None,
                 sample_base: int = 0,
                 gather: Optional[Callable[[torch.Tensor, torch.Tensor], None]] = None,
                 meta: str = "f32"):
        if (avg_bits is None) == (bits is None):
            raise ValueError("give exactly one of avg_bits / bits")
        if meta not in ("f32", "bf16"):
            raise ValueError(f"unknown metadata format {meta!r}")
        self.lib = _lib.load()
        # metadata format: fp32 (zmin, scale) or the paper's bf16 words (NEXT-1)
        self.meta = meta
        self.qfn = self.lib.actnn_quantize if meta == "f32" else self.lib.actnn_quantize_bf16meta
        self.dfn = (self.lib.actnn_dequantize if meta == "f32"
                    else self.lib.actnn_dequantize_bf16meta)
        self.mixed = avg_bits is not None
        self.level_mask = level_mask
        # k > 1: gather(S_global, S_local) fills S_global[N_total] with every
        # rank's S_n (an all-gather over NCCL: the exchange step, equivalent
        # to the all-reduce of zero-padded vectors and exact)
        self.gather = gather
        self.layers: List[Layer] = []
        self.sample_base = sample_base
        lib = self.lib
        for x, seed in zip(xs, seeds):
            x2 = x.reshape(x.shape[0], -1)
            N, D = x2.shape
            nt = n_total if n_total is not None else N
            if self.mixed and nt != N and gather is None:
                # the global S vector would hold only zeros: the allocation
                # needs every rank's S_n (the exchange step)
                raise ValueError("n_total != N (a shard of a larger batch) needs gather= to "
                                 "exchange the per-sample S_n across ranks")
            ng = ceil_div(D, G)
            dev = x2.device
            dt = F32 if x2.dtype == torch.float32 else BF16
            budget = int(avg_bits * nt) if self.mixed else bits * nt
            L = Layer(x2, N, D, ng, dt, seed, budget)
            unit = ng * G // 8
            # Sum_n b_n <= budget globally, so this rank's slice needs at most
            # min(8 N, budget) * unit bytes.
            cap = min(8 * N, budget) * unit
            L.packed = torch.empty(max(cap, 16), dtype=torch.uint8, device=dev)
            if meta == "f32":
                L.zmin = torch.empty(N * ng, dtype=torch.float32, device=dev)
                L.scale = torch.empty(N * ng, dtype=torch.float32, device=dev)
                mq = (_p(L.zmin), _p(L.scale))
            else:
                L.meta = torch.empty(N * ng, dtype=torch.int32, device=dev)
                mq = (_p(L.meta),)
            L.bits = torch.empty(nt, dtype=torch.uint8, device=dev)
            L.off = torch.empty(nt + 1, dtype=torch.int64, device=dev)
            lo = sample_base if nt != N else 0
            bits_p, off_p = _p(L.bits, lo), _p(L.off, lo)
            if self.mixed:
                L.gmin = torch.empty(N * ng, dtype=torch.float32, device=dev)
                L.gmax = torch.empty(N * ng, dtype=torch.float32, device=dev)
                L.S = torch.zeros(nt, dtype=torch.float64, device=dev)
                L.S_loc = (torch.zeros(N, dtype=torch.float64, device=dev) if nt != N
                           else L.S)
                wsb = int(lib.actnn_workspace_bytes(OP_GROUP_STATS, N, D, G))
                L.ws = torch.zeros(max(wsb, 8), dtype=torch.uint8, device=dev)
                L.args["stats"] = (_p(x2), dt, N, D, G, _p(L.gmin), _p(L.gmax), _p(L.S_loc),
                                   _p(L.ws), L.ws.numel())
                L.args["alloc"] = (_p(L.S), None, nt, budget, level_mask, D, G, _p(L.bits),
                                   _p(L.off), None, 0)
                L.args["quant"] = (_p(x2), dt, N, D, G, bits_p, off_p, ctypes.c_uint64(seed),
                                   sample_base, _p(L.gmin), _p(L.gmax), _p(L.packed)) + mq
            else:
                # L2: fixed widths, written once (not part of a step)
                _lib.check(lib.actnn_uniform_bits(nt, D, G, bits, _p(L.bits), _p(L.off),
                                                  _P(torch.cuda.current_stream(dev).cuda_stream)))
                L.args["quant"] = (_p(x2), dt, N, D, G, bits_p, off_p, ctypes.c_uint64(seed),
                                   sample_base, None, None, _p(L.packed)) + mq
            L.args["dequant"] = (_p(L.packed),) + mq + (bits_p, off_p, N, D, G)
            self.layers.append(L)

    # launches per step: stats (K1 with K1b fused) + allocate + quantize + dequantize
    def launches_per_step(self) -> int:
        return len(self.layers) * (4 if self.mixed else 2)

    def compress_layer(self, i: int, stream: ctypes.c_void_p, ev=None):
        lib, L = self.lib, self.layers[i]
        if self.mixed:
            if ev is not None:
                ev[0].record()
            _lib.check(lib.actnn_group_stats(*L.args["stats"], stream))
            if ev is not None:
                ev[1].record()
            if self.gather is not None:
                self.gather(L.S, L.S_loc)
            _lib.check(lib.actnn_allocate_bits(*L.args["alloc"], stream))
        if ev is not None:
            ev[2].record()
        _lib.check(self.qfn(*L.args["quant"], stream))
        if ev is not None:
            ev[3].record()

    def decompress_layer(self, i: int, out: torch.Tensor, out_dt: int, stream, ev=None):
        L = self.layers[i]
        if ev is not None:
            ev[0].record()
        _lib.check(self.dfn(*L.args["dequant"], _p(out), out_dt, stream))
        if ev is not None:
            ev[1].record()

    # ------------------------------------------------------------ pipelined set
    def _events(self):
        if getattr(self, "_evs", None) is None:
            self._evs = [torch.cuda.Event() for _ in self.layers]
        return self._evs

    def compress_all(self, main: torch.cuda.Stream, side: torch.cuda.Stream,
                     alloc: Optional[torch.cuda.Stream] = None,
                     quant2=None, side2=None):
        """Compress every tensor, software-pipelined over streams: the stats
        kernels run back to back on `side`; tensor l's [all-gather ->]
        allocation runs on `alloc` (high priority) once its stats are done, and
        `main` quantises tensor l once its allocation is done.  The single-CTA
        allocator and every kernel's ramp-up/tail overlap other tensors' work.
        `quant2` / `side2` (a stream or a list of streams): the quantisations /
        statistics alternate over main + quant2 / side + side2, so one tensor's
        tail overlaps the next one's ramp-up, as in decompress_all.  Every
        output is ready on `main` on return."""
        if not self.mixed:
            sp = _P(main.cuda_stream)
            for i in range(len(self.layers)):
                _lib.check(self.qfn(*self.layers[i].args["quant"], sp))
            return
        lib = self.lib
        if getattr(self, "_evs2", None) is None:
            self._evs2 = [(torch.cuda.Event(), torch.cuda.Event()) for _ in self.layers]
        alloc = alloc if alloc is not None else side
        def as_list(v):
            return [] if v is None else (list(v) if isinstance(v, (list, tuple)) else [v])

        sides = [side] if alloc is side else [side] + as_list(side2)
        for st in sides:
            st.wait_stream(main)
        ss = [_P(st.cuda_stream) for st in sides]
        sa = _P(alloc.cuda_stream)
        for i, L in enumerate(self.layers):
            ev_stats, ev_alloc = self._evs2[i]
            st = sides[i % len(sides)]
            _lib.check(lib.actnn_group_stats(*L.args["stats"], ss[i % len(sides)]))
            if alloc is not side:
                ev_stats.record(st)
                alloc.wait_event(ev_stats)
            if self.gather is not None:
                with torch.cuda.stream(alloc):
                    self.gather(L.S, L.S_loc)
            _lib.check(lib.actnn_allocate_bits(*L.args["alloc"], sa))
            ev_alloc.record(alloc)
        qs = [main] + as_list(quant2)
        for q in qs[1:]:
            q.wait_stream(main)
        sps = [_P(q.cuda_stream) for q in qs]
        for i, L in enumerate(self.layers):
            qs[i % len(qs)].wait_event(self._evs2[i][1])
            _lib.check(self.qfn(*L.args["quant"], sps[i % len(qs)]))
        for q in qs[1:]:
            main.wait_stream(q)

    def decompress_all(self, outs: Sequence[torch.Tensor], out_dt: int,
                       streams: Sequence[torch.cuda.Stream]):
        """Decompress every tensor into outs[i % len(outs)], alternating streams
        so that one tensor's tail overlaps the next one's ramp-up; streams[0]
        waits for the others on return."""
        k = len(streams)
        for s in streams[1:]:
            s.wait_stream(streams[0])
        sps = [_P(s.cuda_stream) for s in streams]
        for i, L in enumerate(self.layers):
            _lib.check(self.dfn(*L.args["dequant"], _p(outs[i % len(outs)]), out_dt,
                                sps[i % k]))
        for s in streams[1:]:
            streams[0].wait_stream(s)

    def bits_host(self):
        lo = self.sample_base
        return [L.bits[lo:lo + L.N].cpu() if L.bits.numel() != L.N else L.bits.cpu()
                for L in self.layers]


class PipelinedStep:
    """One step of the whole hot path over an ActivationSetPlan -- compress
    every tensor, then decompress every tensor -- in the schedule bench.py
    times: statistics alternating over `n_stats` streams, each tensor's
    [exchange ->] allocation on a high-priority stream, quantisation
    alternating over `n_quant` streams, decompression over `n_dq` streams
    (output buffer i % len(outs)).  `capture()` records the step into one CUDA
    graph (every kernel still runs on each replay); `__call__` replays it, or
    runs the step eagerly when no graph was captured.  The parity tests build
    the same object, so what they check is the launch configuration the bench
    times."""

    def __init__(self, plan: ActivationSetPlan, outs: Sequence[torch.Tensor], out_dt: int,
                 device=None, n_stats: int = 2, n_quant: int = 2, n_dq: int = 3):
        self.plan, self.outs, self.out_dt = plan, list(outs), out_dt
        dev = torch.device(device) if device is not None else plan.layers[0].x.device
        # main: a non-default stream so that the step can be captured
        self.stream = torch.cuda.Stream(dev)
        self.side = torch.cuda.Stream(dev)                    # statistics chain
        self.alloc = torch.cuda.Stream(dev, priority=-1)      # per-tensor allocation
        self.side2 = [torch.cuda.Stream(dev) for _ in range(max(1, n_stats) - 1)]
        self.quant2 = [torch.cuda.Stream(dev) for _ in range(max(1, n_quant) - 1)]
        self.dq = [self.stream] + [torch.cuda.Stream(dev) for _ in range(max(1, n_dq) - 1)]
        self.graph = None

    def compress(self):
        self.plan.compress_all(self.stream, self.side, self.alloc, self.quant2, self.side2)

    def decompress(self):
        self.plan.decompress_all(self.outs, self.out_dt, self.dq)

    def eager(self):
        self.compress()
        self.decompress()

    def capture(self, check_exchange: bool = False):
        """Capture the step into a CUDA graph and replay it once.  With
        `check_exchange` (a multi-rank plan), S is cleared before that replay
        and the replayed widths must equal the eager ones: the captured
        collectives really ran.  Raises on failure (the caller may fall back
        to eager steps)."""
        ref_bits = [L.bits.clone() for L in self.plan.layers] if check_exchange else None
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            self.eager()
        if check_exchange:
            for L in self.plan.layers:
                L.S.zero_()
            torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        if check_exchange and not all(torch.equal(L.bits, r)
                                      for L, r in zip(self.plan.layers, ref_bits)):
            raise RuntimeError("graph replay did not reproduce the eager widths "
                               "(captured exchange not replayed)")
        self.graph = g

    def __call__(self):
        # CUDAGraph.replay() launches on the current stream: make it the main one
        with torch.cuda.stream(self.stream):
            if self.graph is not None:
                self.graph.replay()
            else:
                self.eager()
