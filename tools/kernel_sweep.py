"""Times K1/K3/K4 on a few C3 tensors (CUDA events, median of 10) for the
library loaded by tools/with_variant.py (or the default build).  Diagnostics only."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402

layers = [int(v) for v in os.environ.get("SWEEP_LAYERS", "1,20,60,100").split(",")]
wl = W.workload(os.environ.get("SWEEP_CONFIG", "c3"))
dev = torch.device("cuda:0")
res = {"lib": os.path.basename(A.library_path())}
for li in layers:
    act = wl.acts[li]
    x = W.synth_activation(act, wl.N, li, wl.dtype, dev)
    gmin, gmax, S = A.group_stats(x)
    bits, off = A.allocate_bits(S, int((wl.avg_bits or 2) * wl.N), act.D)
    p = A.quantize(x, bits, off, 7, 0, gmin, gmax)
    out = A.dequantize(p)
    torch.cuda.synchronize()

    def t(fn, reps=10):
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)  # ~1 ms: the launch is queued before the GPU reaches it
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        return ts[len(ts) // 2]

    nbytes = x.numel() * x.element_size()
    tq = t(lambda: A.quantize(x, bits, off, 7, 0, gmin, gmax, packed=p.packed, zmin=p.zmin,
                              scale=p.scale))
    td = t(lambda: A.dequantize(p, out=out))
    ts = t(lambda: A.group_stats(x))
    gn = A.grad_sqnorm(x)
    tg = t(lambda: A.grad_sqnorm(x, out=gn))
    res[f"L{li}"] = {"MB": round(nbytes / 1e6, 1), "stats_us": round(ts, 1),
                     "quant_us": round(tq, 1), "dequant_us": round(td, 1), "sqnorm_us": round(tg, 1),
                     "quant_TBps_in": round(nbytes / tq / 1e6, 2)}
print(json.dumps(res))
