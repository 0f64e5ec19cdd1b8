"""Kernel timeline of the pipelined step (stream-overlap evidence without nsys,
which this image lacks): torch.profiler (Kineto / CUPTI activity records) around
one eager step and one CUDA-graph replay of the exact schedule bench.py times
(plan.PipelinedStep), then a summary from the kernel records:

  * the step's span, the kernels per type (K1 stats, K2 allocation, K3 quantise,
    K4 dequantise, NCCL) with their summed durations and the streams they ran on;
  * concurrency: the fraction of the span with 0 / 1 / 2 / >= 3 kernels resident,
    and how much of each type's time overlaps a kernel of another type (e.g. K1 of
    tensor t + 1 beside K3 of tensor t), i.e. what the multi-stream schedule buys
    over the serial sum.

    python tools/step_timeline.py [--config c3] [--dist] [--trace out.json]

--dist: the multi-rank code path at world size 1 (NCCL process group, the
per-tensor all-gather of S on the high-priority allocation stream, captured in
the graph), as bench.py's ACTNN_FORCE_DIST=1.
"""
import argparse
import gzip
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2104_14129_b200 as A  # noqa: E402
from paper_2104_14129_b200 import dist as AD  # noqa: E402
from paper_2104_14129_b200 import workloads as W  # noqa: E402
from paper_2104_14129_b200.plan import ActivationSetPlan, PipelinedStep  # noqa: E402

TYPES = [("group_stats", "K1"), ("allocate", "K2"), ("dequantize", "K4"),
         ("quantize", "K3"), ("nccl", "NCCL")]


def ktype(name):
    n = name.lower()
    for key, t in TYPES:
        if key in n:
            return t
    return "other"


def kernels_of(trace_path):
    with open(trace_path) as f:
        tr = json.load(f)
    ks = []
    for e in tr.get("traceEvents", []):
        cat = e.get("cat")
        if cat in ("kernel", "Kernel", "gpu_memcpy", "gpu_memset") and e.get("ph") == "X":
            t = ktype(e["name"]) if cat.lower() == "kernel" else cat
            ks.append({"name": e["name"], "t": t, "ts": float(e["ts"]),
                       "dur": float(e["dur"]),
                       "stream": e.get("args", {}).get("stream", e.get("tid"))})
    ks.sort(key=lambda k: k["ts"])
    return ks


def summarise(ks):
    if not ks:
        return {"kernels": 0}
    t0 = min(k["ts"] for k in ks)
    t1 = max(k["ts"] + k["dur"] for k in ks)
    span = t1 - t0
    # sweep: time with c kernels resident, and per type the time it overlaps
    # a kernel of another type
    ev = []
    for i, k in enumerate(ks):
        ev.append((k["ts"], 1, i))
        ev.append((k["ts"] + k["dur"], -1, i))
    ev.sort(key=lambda e: (e[0], e[1]))
    active = set()
    conc = {}
    over = {}
    busy = {}
    last = t0
    for t, d, i in ev:
        dt = t - last
        if dt > 0:
            c = len(active)
            conc[min(c, 3)] = conc.get(min(c, 3), 0.0) + dt
            types = [ks[j]["t"] for j in active]
            for ty in set(types):
                busy[ty] = busy.get(ty, 0.0) + dt
                if any(o != ty for o in types):
                    over[ty] = over.get(ty, 0.0) + dt
        last = t
        if d > 0:
            active.add(i)
        else:
            active.discard(i)
    per = {}
    for k in ks:
        p = per.setdefault(k["t"], {"launches": 0, "sum_dur_us": 0.0, "streams": set()})
        p["launches"] += 1
        p["sum_dur_us"] += k["dur"]
        p["streams"].add(str(k["stream"]))
    for ty, p in per.items():
        # graph replays run each node on an internal stream: report the count
        p["streams"] = len(p["streams"])
        p["sum_dur_us"] = round(p["sum_dur_us"], 1)
        p["busy_us"] = round(busy.get(ty, 0.0), 1)  # union of its launches
        p["overlapped_by_other_types_us"] = round(over.get(ty, 0.0), 1)
        p["overlap_frac"] = round(over.get(ty, 0.0) / max(busy.get(ty, 1e-9), 1e-9), 3)
    serial = sum(k["dur"] for k in ks)
    phases = {}
    for name, tys in (("compress", ("K1", "K2", "K3", "NCCL", "gpu_memcpy")), ("decompress", ("K4",))):
        sel = [k for k in ks if k["t"] in tys]
        if sel:
            a = min(k["ts"] for k in sel)
            b = max(k["ts"] + k["dur"] for k in sel)
            phases[name] = {"start_us": round(a - t0, 1), "end_us": round(b - t0, 1),
                            "span_us": round(b - a, 1)}
    return {"phases": phases, "kernels": len(ks), "span_us": round(span, 1),
            "serial_sum_us": round(serial, 1),
            "serial_sum_over_span": round(serial / span, 3),
            "time_frac_with_n_kernels": {("3+" if c == 3 else str(c)): round(v / span, 3)
                                         for c, v in sorted(conc.items())},
            "per_type": per}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--dist", action="store_true")
    ap.add_argument("--trace", default=None, help="keep the graph-replay trace (gzip json)")
    args = ap.parse_args()

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    gather = None
    if args.dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29571")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
        gather = AD.make_gather(1, "nccl")
    wl = W.workload(args.config)
    xs = [W.synth_activation(a, wl.N, t, wl.dtype, dev) for t, a in enumerate(wl.acts)]
    torch.cuda.synchronize()
    plan = ActivationSetPlan(xs, [W.quant_seed(t) for t in range(len(wl.acts))],
                             avg_bits=wl.avg_bits, bits=None if wl.avg_bits else wl.bits,
                             n_total=wl.N, sample_base=0, gather=gather)
    tdt = torch.float32 if wl.dtype == "f32" else torch.bfloat16
    mx = max(x.numel() for x in xs)
    outs = [torch.empty(mx, dtype=tdt, device=dev) for _ in range(3)]
    out_dt = A.api.F32 if wl.dtype == "f32" else A.api.BF16
    ps = PipelinedStep(plan, outs, out_dt, dev)
    torch.cuda.set_stream(ps.stream)
    for _ in range(3):
        ps()
    torch.cuda.synchronize()

    from torch.profiler import ProfilerActivity, profile
    res = {"config": args.config, "dist_path": bool(args.dist)}
    tmp = tempfile.mkdtemp()
    # eager step (the real streams)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ps()
        torch.cuda.synchronize()
    p_e = os.path.join(tmp, "eager.json")
    prof.export_chrome_trace(p_e)
    res["eager"] = summarise(kernels_of(p_e))
    # graph replay (what bench.py times)
    ps.capture(check_exchange=args.dist)
    for _ in range(2):
        ps()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ps()
        torch.cuda.synchronize()
    p_g = os.path.join(tmp, "graph.json")
    prof.export_chrome_trace(p_g)
    res["graph"] = summarise(kernels_of(p_g))
    # the same step unprofiled, for comparison with the traced span
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        ps()
    b.record()
    torch.cuda.synchronize()
    res["graph_step_ms_unprofiled"] = round(a.elapsed_time(b) / 5, 3)
    if args.trace:
        ks = kernels_of(p_g)
        with gzip.open(args.trace, "wt") as f:
            json.dump([[k["t"], k["stream"], round(k["ts"], 2), round(k["dur"], 2)] for k in ks], f)
    print(json.dumps(res))
    if args.dist:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
