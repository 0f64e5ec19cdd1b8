"""One whole pipelined C3 step inside a cudaProfilerStart/Stop range, for
   ncu --replay-mode app-range --profile-from-start off \
       --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
       python tools/step_dram.py [--graph]
which reports the DRAM bytes the whole step moved (measured
bytes vs the 70.4 GB algorithmic figure).  Not a bench: no number taken under
a profiler is reported as a bench value."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402
from paper_2104_14129_b200.plan import ActivationSetPlan, PipelinedStep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--graph", action="store_true")
a = ap.parse_args()
wl = W.workload(a.config)
dev = torch.device("cuda:0")
xs = [W.synth_activation(x, wl.N, t, wl.dtype, dev) for t, x in enumerate(wl.acts)]
plan = ActivationSetPlan(xs, [W.quant_seed(t) for t in range(len(xs))], avg_bits=wl.avg_bits,
                         bits=None if wl.avg_bits else wl.bits)
tdt = xs[0].dtype
outs = [torch.empty(max(x.numel() for x in xs), dtype=tdt, device=dev) for _ in range(3)]
ps = PipelinedStep(plan, outs, A.api.F32 if wl.dtype == "f32" else A.api.BF16)
torch.cuda.set_stream(ps.stream)
for _ in range(2):
    ps()
if a.graph:
    ps.capture()
torch.cuda.synchronize()
bits = [L.bits[:L.N].cpu() for L in plan.layers]
alg = 0
s = xs[0].element_size()
for L, b in zip(plan.layers, bits):
    g = L.N * L.ng
    packed = int(b.long().sum()) * L.ng * 32
    alg += 2 * L.N * L.D * s + 8 * g + 8 * g + packed + 8 * g + 8 * L.N * (-(-L.ng // 32))  # stats + quantise
    alg += packed + 8 * g + L.N * L.D * s                                                 # dequantise
print("algorithmic_bytes_per_step", alg, flush=True)
torch.cuda.cudart().cudaProfilerStart()
ps()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
