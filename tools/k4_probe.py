"""K4 timing probe (diagnostics): dequantize of every C3 tensor back to back
(one event pair per launch, as bench.py's breakdown) and of the largest tensor
alone, for the library loaded by tools/with_variant.py."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402

cfg = os.environ.get("PROBE_CONFIG", "c3")
wl = W.workload(cfg)
dev = torch.device("cuda:0")
ps = []
out = None
for li, act in enumerate(wl.acts):
    x = W.synth_activation(act, wl.N, li, wl.dtype, dev)
    p = A.compress(x, seed=W.quant_seed(li), avg_bits=wl.avg_bits)
    n = int(p.off[-1].item())
    p.packed = p.packed[:max(n, 16)].clone()
    ps.append((p, x.numel(), x.element_size()))
    del x
    torch.cuda.synchronize()
mx = max(n for _, n, _ in ps)
out = torch.empty(mx, dtype=torch.float32 if wl.dtype == "f32" else torch.bfloat16, device=dev)


def run_all(evs):
    for (p, n, s), (a, b) in zip(ps, evs):
        a.record()
        A.dequantize(p, out=out[:n].view(p.shape))
        b.record()


evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for _ in ps] for _ in range(4)]
run_all(evs[0])
torch.cuda.synchronize()
tot = []
per = [0.0] * len(ps)
for r in range(1, 4):
    torch.cuda._sleep(50_000_000)
    run_all(evs[r])
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in evs[r]]
    tot.append(sum(ts))
    per = [q + t / 3 for q, t in zip(per, ts)]
alg = sum(int(p.off[-1].item()) + 8 * p.zmin.numel() + 9 * p.N + n * s for p, n, s in ps)
big = max(range(len(ps)), key=lambda i: ps[i][1])
pb, nb, sb = ps[big]
algb = int(pb.off[-1].item()) + 8 * pb.zmin.numel() + 9 * pb.N + nb * sb
res = {"config": cfg, "serial_ms": min(tot), "GBps_alg": alg / (min(tot) * 1e-3) / 1e9,
       "largest_us": per[big] * 1e3, "largest_GBps": algb / (per[big] * 1e-3) / 1e9,
       "small_share": sum(t for t, (_, n, s) in zip(per, ps) if n * s < 120e6) / sum(per),
       "small_ms": sum(t for t, (_, n, s) in zip(per, ps) if n * s < 120e6),
       "large_ms": sum(t for t, (_, n, s) in zip(per, ps) if n * s >= 120e6)}
if os.environ.get("PROBE_DUMP"):
    res["layers"] = [[n * s, int(p.off[-1].item()) + 8 * p.zmin.numel() + 9 * p.N + n * s,
                      round(t * 1e3, 2)] for (p, n, s), t in zip(ps, per)]
print(json.dumps(res))

# per size class: 8 back-to-back launches of one tensor of the class between one
# event pair (no per-launch event overhead), best of 3
if os.environ.get("PROBE_SIZES"):
    seen = {}
    for i, (p, n, s) in enumerate(ps):
        seen.setdefault(n * s, i)
    rows = []
    for nbytes, i in sorted(seen.items()):
        p, n, s = ps[i]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            torch.cuda._sleep(20_000_000)
            a.record()
            for _ in range(8):
                A.dequantize(p, out=out[:n].view(p.shape))
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 8)
        algi = int(p.off[-1].item()) + 8 * p.zmin.numel() + 9 * p.N + n * s
        rows.append([round(nbytes / 1e6, 1), sum(1 for _, m, t in ps if m * t == nbytes),
                     round(best * 1e3, 1), round(algi / (best * 1e-3) / 1e9)])
    print(json.dumps({"config": cfg, "sizes_MB_count_us_GBps": rows}))
