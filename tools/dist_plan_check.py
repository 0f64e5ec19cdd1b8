"""Two ranks on one GPU (gloo; NCCL refuses two ranks per device) driving the
product's multi-rank path -- ActivationSetPlan with the exchange closure of
dist.make_gather, issued through plan.PipelinedStep (compress_all: stats ->
all-gather of S on the allocation stream -> allocation -> quantise; then
decompress_all) -- against the oracle's sharded driver O13 (SURVEY §8(c),
§8(e)).  Run by tests/test_gpu_dist.py:
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_plan_check.py
Prints "OK" on rank 0 when every rank's widths, packed bytes, zmin, scale and
dequantised values equal the oracle's for that rank."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle as O
    import paper_2104_14129_b200 as A
    from paper_2104_14129_b200 import dist as AD
    from paper_2104_14129_b200 import workloads as W
    from paper_2104_14129_b200.plan import ActivationSetPlan, PipelinedStep

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    acts = [a for i, a in enumerate(W.resnet_activation_set(50)) if i in (0, 5, 40, 100, 106)]
    n_tot, avg = 16, 2.0
    lo, hi = AD.shard_range(n_tot, rank, world)
    full = [W.synth_activation(a, n_tot, t, "f32", dev) for t, a in enumerate(acts)]
    xs = [f[lo:hi].contiguous() for f in full]
    seeds = [W.quant_seed(t) for t in range(len(acts))]
    plan = ActivationSetPlan(xs, seeds, avg_bits=avg, n_total=n_tot, sample_base=lo,
                             gather=AD.make_gather(world, "gloo"))
    outs = [torch.empty(x.numel(), dtype=torch.float32, device=dev) for x in xs]
    ps = PipelinedStep(plan, outs, A.api.F32)
    torch.cuda.set_stream(ps.stream)
    ps()
    torch.cuda.synchronize()
    mine = []
    for L, o in zip(plan.layers, outs):
        off = L.off[lo:hi + 1].cpu().numpy()
        nb = int(off[-1] - off[0])
        mine.append((L.bits[lo:hi].cpu().numpy(), L.packed[:nb].cpu().numpy(),
                     L.zmin.cpu().numpy(), L.scale.cpu().numpy(), o.cpu().numpy()))
    got = [None] * world
    dist.all_gather_object(got, mine)
    if rank == 0:
        for t, (a, f) in enumerate(zip(acts, full)):
            xh = f.cpu().numpy().reshape(n_tot, -1)
            ref = O.sharded_quantize(xh, world, avg, seeds[t], threads=8)
            for r in range(world):
                bits, packed, zmin, scale, out = got[r][t]
                rp, rz, rs, rb = ref[r]
                assert np.array_equal(bits, rb), (t, r, "bits")
                assert np.array_equal(packed, rp), (t, r, "packed")
                assert np.array_equal(zmin.view(np.uint32), rz.ravel().view(np.uint32)), (t, r)
                assert np.array_equal(scale.view(np.uint32), rs.ravel().view(np.uint32)), (t, r)
                exp = O.dequantize(rp, rz, rs, rb, len(rb), a.D)
                assert np.array_equal(out.view(np.uint32), exp.ravel().view(np.uint32)), (t, r)
        print("OK: %d ranks x %d tensors equal the oracle's sharded driver" % (world, len(acts)))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
