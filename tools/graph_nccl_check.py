"""Graph capture of the pipelined step with an NCCL all-gather of S (1-rank
group): replays must equal the eager step byte for byte.  Run by
tests/test_gpu_parity.py in a fresh process; prints OK."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402
from paper_2104_14129_b200.plan import ActivationSetPlan  # noqa: E402

DEV = torch.device("cuda:0")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29547")
torch.cuda.set_device(DEV)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
try:
    acts = [W.resnet_activation_set(50)[i] for i in (3, 12, 40)]
    xs = [W.synth_activation(a, 8, i, "f32", DEV) for i, a in enumerate(acts)]

    def gather(S, S_loc):
        dist.all_gather_into_tensor(S, S_loc)

    plan = ActivationSetPlan(xs, [11, 12, 13], avg_bits=2.0, n_total=8, gather=gather)
    outs = [torch.empty(max(x.numel() for x in xs), device=DEV) for _ in range(2)]
    main, side, al, aux = (torch.cuda.Stream(), torch.cuda.Stream(),
                           torch.cuda.Stream(priority=-1), torch.cuda.Stream())
    with torch.cuda.stream(main):
        plan.compress_all(main, side, al)
        plan.decompress_all(outs, A.api.F32, [main, aux])
    torch.cuda.synchronize()
    ref = [L.packed.cpu().numpy().copy() for L in plan.layers]
    ref_bits = [L.bits.cpu().numpy().copy() for L in plan.layers]
    ref_out = outs[0].cpu().numpy().copy()
    for L in plan.layers:
        L.packed.zero_()
        L.S.zero_()
    outs[0].zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        plan.compress_all(main, side, al)
        plan.decompress_all(outs, A.api.F32, [main, aux])
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for L, r, rb in zip(plan.layers, ref, ref_bits):
        assert np.array_equal(L.bits.cpu().numpy(), rb), "bits"
        assert np.array_equal(L.packed.cpu().numpy(), r), "packed"
    assert np.array_equal(outs[0].cpu().numpy(), ref_out), "dequantized"
    print("OK")
finally:
    dist.destroy_process_group()
