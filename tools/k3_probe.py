"""K3 timing probe (diagnostics): the mixed-path quantiser of every tensor of a
set back to back (one event pair per launch, as bench.py's breakdown), with
statistics and widths precomputed, for the library loaded by
tools/with_variant.py.  PROBE_CONFIG = c3 | c4 | c2 (c2: single pass)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402

cfg = os.environ.get("PROBE_CONFIG", "c4")
wl = W.workload(cfg)
dev = torch.device("cuda:0")
items = []
for li, act in enumerate(wl.acts):
    x = W.synth_activation(act, wl.N, li, wl.dtype, dev)
    if wl.avg_bits is not None:
        gmin, gmax, S = A.group_stats(x)
        bits, off = A.allocate_bits(S, int(wl.avg_bits * wl.N), act.D)
    else:
        gmin = gmax = None
        bits, off = A.uniform_bits(wl.N, act.D, wl.bits, dev)
    p = A.quantize(x, bits, off, W.quant_seed(li), 0, gmin, gmax)
    items.append((x, bits, off, gmin, gmax, p))
torch.cuda.synchronize()


def run_all(evs):
    for (x, bits, off, gmin, gmax, p), (a, b) in zip(items, evs):
        a.record()
        A.quantize(x, bits, off, 7, 0, gmin, gmax, packed=p.packed, zmin=p.zmin, scale=p.scale)
        b.record()


evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for _ in items] for _ in range(4)]
run_all(evs[0])
torch.cuda.synchronize()
tot, per = [], [0.0] * len(items)
for r in range(1, 4):
    torch.cuda._sleep(100_000_000)
    run_all(evs[r])
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in evs[r]]
    tot.append(sum(ts))
    per = [q + t / 3 for q, t in zip(per, ts)]


def alg(it):
    x, bits, off, gmin, gmax, p = it
    E = x.numel()
    groups = p.zmin.numel()
    mm = 8 * groups if gmin is not None else 0
    return E * x.element_size() + mm + int(off[-1].item()) + 8 * groups + 9 * x.shape[0]


al = [alg(it) for it in items]
big = max(range(len(items)), key=lambda i: items[i][0].numel())
res = {"config": cfg, "serial_ms": round(min(tot), 3),
       "GBps_alg": round(sum(al) / (min(tot) * 1e-3) / 1e9, 1),
       "largest_us": round(per[big] * 1e3, 1),
       "largest_GBps": round(al[big] / (per[big] * 1e-3) / 1e9, 1)}
print(json.dumps(res))
