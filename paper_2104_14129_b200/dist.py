"""Batch-sharded (data-parallel) compression across ranks -- SURVEY §8(e).

Samples are the independent units of the method: quantising sample n touches
only sample n's groups, width and offset, and its Philox counters use the
GLOBAL element index e = (sample_base + n) * D + d, so results do not depend on
where a sample lives.  The one coupling is the per-layer allocation (P:558:
"computes the optimal b_n for each sample under a fixed bits budget for this
layer"), which here is global over the whole batch: every rank computes its
samples' S_n, the S vector is exchanged (the only collective of the path, one
per tensor, <= 32 KB), and every rank runs the same deterministic allocator on
the full vector and keeps its own slice of the widths/offsets.  The k-rank
output, concatenated in rank order, is byte-identical to the 1-rank output
(tests/test_dist_gloo.py, tests/test_gpu_parity.py::test_virtual_ranks_*).

The collective goes through torch.distributed (NCCL over NVLink on B200s, gloo
for the CPU tests).  This module holds plumbing only: shard arithmetic and the
exchange.  All arithmetic of the method runs in libactnn.so.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous batch slice [lo, hi) of `rank`; equal slices required."""
    if n_total % world:
        raise ValueError(f"batch {n_total} is not divisible by world size {world}")
    n = n_total // world
    return rank * n, (rank + 1) * n


def allreduce_sens(S_padded: torch.Tensor, group=None) -> torch.Tensor:
    """Sum of the ranks' zero-padded S vectors (exact: x + 0 = x)."""
    dist.all_reduce(S_padded, op=dist.ReduceOp.SUM, group=group)
    return S_padded


def gather_sens(S_global: torch.Tensor, S_local: torch.Tensor, group=None) -> None:
    """S_global[r*n:(r+1)*n] = rank r's S_local (the same exchange as the
    zero-padded all-reduce, with a quarter of the bytes for k = 4)."""
    dist.all_gather_into_tensor(S_global, S_local, group=group)


def make_gather(world: int, backend: str = "nccl", group=None):
    """The exchange step as the closure ActivationSetPlan calls per tensor:
    gather(S_global, S_local) fills S_global[r*n:(r+1)*n] with rank r's S_n.

    north_star names "an NCCL all-reduce of the allocator statistics"; the
    all-gather is the same exchange (every rank ends with the identical global
    S vector, bit for bit, since the zero-padded sum adds only exact zeros;
    tests/test_dist_gloo.py checks the two agree) with 1/k of the bytes and no
    per-step clearing of the padded vector.  NCCL: all_gather_into_tensor on
    the current stream (capturable in a CUDA graph); gloo (test mode, several
    ranks on one device or CPU): the list form."""
    if backend == "nccl":
        def gather(S_global: torch.Tensor, S_local: torch.Tensor) -> None:
            dist.all_gather_into_tensor(S_global, S_local, group=group)
    else:
        def gather(S_global: torch.Tensor, S_local: torch.Tensor) -> None:
            dist.all_gather(list(S_global.view(world, -1).unbind(0)), S_local, group=group)
    return gather


def local_slice(bits_g: torch.Tensor, off_g: torch.Tensor, lo: int, hi: int):
    """This rank's widths and offsets.  The ABI addresses sample n at
    packed + off[n] - off[0], so the slice off_g[lo:hi+1] is used as is."""
    return bits_g[lo:hi], off_g[lo:hi + 1]


def compress_sharded(x_local: torch.Tensor, seed: int, avg_bits: float,
                     group=None, level_mask: Optional[int] = None):
    """One tensor's mixed-precision compress on this rank's batch shard with
    the allocation computed globally (all ranks must call it)."""
    from . import api
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_loc = x_local.shape[0]
    lo, _ = shard_range(n_loc * world, rank, world)
    kw = {} if level_mask is None else {"level_mask": level_mask}
    return api.compress(x_local, seed, avg_bits=avg_bits, sample_base=lo,
                        sens_allreduce=lambda S: allreduce_sens(S, group),
                        n_total=n_loc * world, **kw)
