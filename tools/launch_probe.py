"""Fixed per-launch cost in the serial breakdown pattern (diagnostics): an
event pair around (a) an empty spin kernel, (b) K1 / K3 / K4 on tiny inputs,
each launch queued behind a long spin so host enqueue gaps do not show."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402

dev = torch.device("cuda:0")
x = torch.randn(256, 2048, device=dev).clamp_min_(0)
gmin, gmax, S = A.group_stats(x)
bits, off = A.allocate_bits(S, 512, 2048)
p = A.quantize(x, bits, off, 7, 0, gmin, gmax)
out = A.dequantize(p)
xu = torch.randn(256, 2048, device=dev)
pu = A.compress(xu, seed=3, bits=2)
torch.cuda.synchronize()
fns = {"empty_spin": lambda: torch.cuda._sleep(0),
       "K1_stats_2MB": lambda: A.group_stats(x, sens_out=S),
       "K2_alloc_256": lambda: A.allocate_bits(S, 512, 2048),
       "K3_ws_2MB": lambda: A.quantize(x, bits, off, 7, 0, gmin, gmax, packed=p.packed,
                                       zmin=p.zmin, scale=p.scale),
       "K3_fast_uniform_2MB": lambda: A.quantize(xu, pu.bits, pu.off, 3, 0, packed=pu.packed,
                                                 zmin=pu.zmin, scale=pu.scale),
       "K4_2MB": lambda: A.dequantize(p, out=out)}
res = {}
for name, fn in fns.items():
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(50)]
    torch.cuda._sleep(200_000_000)
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    res[name] = round(ts[len(ts) // 2], 2)
print(json.dumps(res))
