"""Multi-process (world_size 2, gloo, CPU) test of the batch-sharded plumbing
in paper_2104_14129_b200/dist.py: shard ranges, the S exchange (zero-padded
all-reduce and all-gather agree), the global allocation and the per-rank
slices of widths/offsets with sample_base.  The per-rank compute is the CPU
oracle (there is no GPU here); the concatenated per-rank bytes must equal the
1-rank result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, D, avg, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2104_14129_b200 import dist as AD
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        x = (rng.standard_normal((N, D)) * np.exp(rng.standard_normal((N, 1)))).astype(np.float32)
        lo, hi = AD.shard_range(N, rank, world)
        mn, mx = O.group_minmax(x[lo:hi])
        S_loc = torch.from_numpy(O.sensitivity(mn, mx))
        S_pad = torch.zeros(N, dtype=torch.float64)
        S_pad[lo:hi] = S_loc
        S_ar = AD.allreduce_sens(S_pad.clone())
        S_ag = torch.zeros(N, dtype=torch.float64)
        AD.gather_sens(S_ag, S_loc)
        assert torch.equal(S_ar, S_ag)
        # the closure the plan (and bench.py) call per tensor, gloo form
        S_cl = torch.full((N,), -1.0, dtype=torch.float64)
        AD.make_gather(world, "gloo")(S_cl, S_loc)
        assert torch.equal(S_cl, S_ar)
        bits_g = O.allocate_bits(S_ar.numpy(), int(avg * N))
        off_g = O.offsets(bits_g, D)
        b_l, o_l = AD.local_slice(torch.from_numpy(bits_g), torch.from_numpy(off_g), lo, hi)
        packed, zmin, scale, off_l = O.quantize(x[lo:hi], b_l.numpy(), seed, lo)
        assert np.array_equal(o_l.numpy() - o_l[0].item(), off_l)
        out = [None] * world
        dist.all_gather_object(out, (packed.tobytes(), zmin.tobytes(), scale.tobytes(),
                                     b_l.numpy().tobytes()))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_equals_single_rank(world):
    import oracle as O
    N, D, avg, seed = 8, 1024, 2.0, 31
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, D, avg, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((N, D)) * np.exp(rng.standard_normal((N, 1)))).astype(np.float32)
    ref = O.sharded_quantize(x, 1, avg, seed)[0]
    cat = [b"".join(o[i] for o in out) for i in range(4)]
    assert cat[0] == ref[0].tobytes()
    assert cat[1] == ref[1].tobytes() and cat[2] == ref[2].tobytes()
    assert cat[3] == ref[3].tobytes()


def test_shard_range():
    from paper_2104_14129_b200 import dist as AD
    assert AD.shard_range(4096, 3, 8) == (1536, 2048)
    with pytest.raises(ValueError):
        AD.shard_range(10, 0, 4)
