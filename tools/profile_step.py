"""Runs `--steps` steps of the bench workload (after one warm-up step) so that
ncu sees a known launch sequence.  Launch order per step: for every tensor
l: group_stats_kernel, sens_reduce_kernel, allocate_kernel, quantize_fast_kernel
(mixed) then, for every tensor, dequantize_fast_kernel.  Not a bench: numbers
taken under a profiler are never reported as bench values."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2104_14129_b200 import workloads as W  # noqa: E402
from paper_2104_14129_b200.api import BF16, F32  # noqa: E402
from paper_2104_14129_b200.plan import ActivationSetPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--layers", default="")
a = ap.parse_args()
wl = W.workload(a.config)
acts = wl.acts
idx = list(range(len(acts))) if not a.layers else [int(v) for v in a.layers.split(",")]
dev = torch.device("cuda:0")
xs = [W.synth_activation(acts[i], wl.N, i, wl.dtype, dev) for i in idx]
plan = ActivationSetPlan(xs, [W.quant_seed(i) for i in idx], avg_bits=wl.avg_bits,
                         bits=None if wl.avg_bits else wl.bits)
out = torch.empty(max(x.numel() for x in xs), dtype=xs[0].dtype, device=dev)
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
odt = F32 if wl.dtype == "f32" else BF16
for _ in range(1 + a.steps):
    for i in range(len(idx)):
        plan.compress_layer(i, sp)
    for i in range(len(idx)):
        plan.decompress_layer(i, out, odt, sp)
torch.cuda.synchronize()
print("layers", len(idx), "launches/step", plan.launches_per_step())
