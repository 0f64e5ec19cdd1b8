"""Launches the NEXT-3 kernels once each on realistic sizes so that ncu can
capture them: K6 grad_sqnorm on the largest C3 tensor (fp32) and the largest
C4 tensor (bf16), then K5 (stage 2) on the C4 problem (311 layers x 1024
samples).  Not a bench: numbers taken under a profiler are never reported."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402

dev = torch.device("cuda:0")
for cfg in ("c3", "c4"):
    wl = W.workload(cfg)
    x = W.synth_activation(wl.acts[1], wl.N, 1, wl.dtype, dev)
    A.grad_sqnorm(x)
    del x
wl = W.workload("c4")
D = [a.D for a in wl.acts]
g = torch.Generator(device=dev).manual_seed(0)
sens = torch.exp(torch.randn((len(D), wl.N), generator=g, device=dev, dtype=torch.float64))
alloc = A.LayerAllocator(D, wl.N, dev)
alloc(sens, int(1.25 * wl.N * sum(D)))
torch.cuda.synchronize()
print("ok")
