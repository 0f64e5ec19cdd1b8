#!/usr/bin/env python
"""bench.py -- ActNN's hot path (per-group SR compressor + decompressor +
per-sample greedy allocator) on B200, BASELINE.json's metric.

A step = one pass of the whole hot path over one batch: for every tensor of
the activation set, compress (group stats -> [all-gather of S, k > 1] ->
greedy allocation -> SR quantise + pack) and decompress (unpack + dequantise).
Default workload: C3 = the ResNet-50 activation set (107 tensors), batch 256
per GPU, fp32, per-sample widths {1,2,4,8} averaging 2 bits.  Under torchrun
each rank owns 256 samples (weak scaling) and the allocation is global over
all ranks' samples.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c4|c5]
  python bench.py --impl reference ...   # the CPU oracle on a bounded sample

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress+decompress GB/s and % HBM peak at 1/2/4/8 B200; codes bit-exact vs oracle"
FALLBACK_HBM_GBS = 6650.0
NOMINAL_HBM_GBS = 8000.0   # B200 HBM3e nominal ("report both")

# The paper's own numbers nearest to this path, with their hardware (BASELINE.md
# §1).  Context only: the paper publishes no compressor / decompressor throughput.
PAPER_CONTEXT = {
    "note": "PAPER.md reports no compressor/decompressor throughput (BASELINE.json "
            "'published' is empty); these are its end-to-end figures, other hardware, "
            "fp32 PyTorch 1.7 training -- context, not targets",
    "hardware": "1x NVIDIA T4 16 GB (AWS g4dn.4xlarge), 64 GB host, PyTorch 1.7 (P:820)",
    "figures": [
        {"what": "ResNet-152 activation memory, FP -> ActNN L3 (2-bit), batch 32 / 64",
         "value": "5.28 -> 0.44 GB / 10.57 -> 0.88 GB (12x)", "cite": "P:765-766 (Table 4)"},
        {"what": "ResNet-152 total memory, FP -> L3, batch 32 / 64",
         "value": "6.01 -> 1.18 GB / 11.32 -> 1.64 GB", "cite": "P:765-766 (Table 4)"},
        {"what": "bits per element of a Conv-BN-ReLU block (bf16 metadata)",
         "value": "5.25 vs 64 -> 12.19x", "cite": "P:826-828"},
        {"what": "training throughput of the largest ResNet-152 variant at batch 64, "
                 "FP / L3 / L4 (depth, width, resolution scaling)",
         "value": "0.59/0.46/0.38, 0.70/1.07/1.09, 0.59/0.46/0.42 TFLOPS",
         "cite": "P:849-851 (Table 5)"},
    ],
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="actnn", choices=["actnn", "reference"])
    ap.add_argument("--config", default="c3", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--levels", default="pow2", choices=["pow2", "unit"],
                    help="allocator widths: {1,2,4,8} (hot path) or 1..8 (the paper's unit step)")
    ap.add_argument("--meta", default="f32", choices=["f32", "bf16"],
                    help="per-group metadata: fp32 (zmin, scale) or the paper's bf16 words")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-adapt", action="store_true",
                    help="skip the NEXT-3 side measurement (gradient norms, stage-2 allocation)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="replay the step from a captured CUDA graph (default at N=1)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--no-side", action="store_true",
                    help="skip the C2 / C4 side legs of the default (C3, N=1) run")
    ap.add_argument("--side-steps", type=int, default=10)
    ap.add_argument("--pool", type=int, default=0,
                    help="C5 below 4 GPUs: R distinct resident input buffers per tensor shape, "
                         "reused by the tensors of that shape (0: automatic when the whole "
                         "set does not fit)")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key, mixed=True):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel, from
    the committed ncu launch list of one C3 step (profiles/traffic.json)."""
    name = {"stats": "group_stats_kernel",
            "quantize": "quantize_ws_kernel" if mixed else "quantize_fast_kernel",
            "dequantize": "dequantize_fast_kernel"}[kernel_key]
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)["kernels"][name]["dram_bytes_per_launch"]
    except Exception:
        return None


# ------------------------------------------------------------------ clocks
REASONS = [(0x4, "sw_power_cap"), (0x8, "hw_slowdown"), (0x20, "sw_thermal_slowdown"),
           (0x40, "hw_thermal_slowdown"), (0x80, "hw_power_brake_slowdown"),
           (0x2, "applications_clocks_setting"), (0x1, "gpu_idle")]


class ClockSampler:
    """Samples SM clock and clock-event reasons through NVML every 10 ms."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in REASONS:
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# ------------------------------------------------------------------ helpers
def algorithmic_bytes(layers, bits_host, s_in, s_out, mixed, meta_bytes=8):
    """Per-kernel algorithmic bytes (SURVEY §8(d) / DESIGN.md 'Roofline').
    meta_bytes: stored metadata per group (8 fp32, 4 with bf16 words)."""
    tot = {"stats": 0, "quantize": 0, "dequantize": 0}
    for L, b in zip(layers, bits_host):
        groups = L.N * L.ng
        E = L.N * L.D
        packed = int(b.long().sum()) * L.ng * 32
        mm = 8 * groups           # gmin/gmax (K1 -> K3), always fp32
        meta = meta_bytes * groups
        if mixed:
            tot["stats"] += E * s_in + mm + 8 * L.N * (-(-L.ng // 32))
            tot["quantize"] += E * s_in + mm + packed + meta + 9 * L.N
        else:
            tot["quantize"] += E * s_in + packed + meta + 9 * L.N
        tot["dequantize"] += packed + meta + 9 * L.N + E * s_out
    return tot


def cpu_sample(wl, acts, args, target_s, seed_of, torch):
    """Bounded CPU oracle run of the same workload: for every tensor of the
    set, the first n_s samples go through stats -> heap allocation ->
    quantize -> dequantize.  n_s is calibrated so the run takes ~target_s."""
    import numpy as np
    import oracle as O
    from paper_2104_14129_b200 import workloads as W
    cores = os.cpu_count() or 1

    def run(n_s, xs_host):
        t0 = time.perf_counter()
        for li, (a, xh) in enumerate(zip(acts, xs_host)):
            xh = xh[:n_s]
            if wl.avg_bits is not None:
                mn, mx = O.group_minmax(xh)
                S = O.sensitivity(mn, mx)
                bits = O.allocate_bits(S, int(wl.avg_bits * n_s))
            else:
                bits = np.full(n_s, wl.bits, np.uint8)
            packed, zmin, scale, _ = O.quantize(xh, bits, seed_of(li), 0, threads=cores)
            O.dequantize(packed, zmin, scale, bits, n_s, a.D,
                         out_dtype=O.F32 if wl.dtype == "f32" else O.BF16, threads=cores)
        return time.perf_counter() - t0

    def host_inputs(n):
        out = []
        for li, a in enumerate(acts):
            x = W.synth_activation(a, n, li, wl.dtype, "cpu")
            if wl.dtype == "bf16":
                out.append(x.view(torch.int16).numpy().view(np.uint16))
            else:
                out.append(x.numpy())
        return out

    # calibrate: double the sample until one run takes >= target/4, then scale
    n_s, t = 1, 0.0
    while True:
        xs = host_inputs(n_s)
        t = run(n_s, xs)
        if t >= target_s / 4 or n_s >= wl.N:
            break
        n_s = min(wl.N, 2 * n_s)
    n_new = max(1, min(wl.N, int(n_s * target_s / max(t, 1e-3))))
    if n_new > n_s:
        n_s = n_new
        xs = host_inputs(n_s)
        t = run(n_s, xs)
    E = n_s * sum(a.D for a in acts)
    s_in = 4 if wl.dtype == "f32" else 2
    return {"value": E * s_in / t / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"first {n_s} of {wl.N} samples of each of the {len(acts)} tensors "
                      f"({E} elements, {E * s_in / 1e9:.2f} GB in), full compress+decompress "
                      f"(stats, heap allocation, quantize, dequantize), {t:.1f} s"}, t


def config_dict(wl, args, world, n_loc):
    s_in = 4 if wl.dtype == "f32" else 2
    E = n_loc * sum(a.D for a in wl.acts)
    return {
        "workload": f"{wl.name.upper()}: {wl.description}",
        "tensors": len(wl.acts),
        "samples_per_gpu": n_loc,
        "global_batch": n_loc * world,
        "elements_per_gpu_step": E,
        "bytes_in_per_gpu_step": E * s_in,
        "G": 256,
        "bits": ("per-sample %s, avg %.2f (greedy, global over ranks)"
                 % ("1..8 (unit step)" if getattr(args, "levels", "pow2") == "unit"
                    else "{1,2,4,8}", wl.avg_bits))
        if wl.avg_bits is not None else f"uniform {wl.bits}",
        "parallelism": f"dp{world} (batch-sharded; all-gather of S per tensor)" if world > 1
        else "dp1",
        "l2": "inputs larger than L2: %.1f GB per step per GPU vs 126 MB L2" % (E * s_in / 1e9),
        "cuda_graph": bool(getattr(args, "graph", False)),
        "metadata": ("bf16 (Z', R') word per group, 0.125 bits/elem (P:513)"
                     if getattr(args, "meta", "f32") == "bf16"
                     else "fp32 (zmin, scale) per group, 0.25 bits/elem"),
    }


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    import torch
    from paper_2104_14129_b200 import workloads as W
    wl = W.workload(args.config)
    world = args.gpus
    n_loc = wl.N // world if args.config == "c5" else wl.N
    per_step = max(1.0, min(5.0, 150.0 / max(1, args.steps + args.warmup)))
    cb, _ = cpu_sample(wl, wl.acts, args, per_step, W.quant_seed, torch)
    # steps: the same bounded sample, timed again K times after W warm-ups
    import numpy as np
    import oracle as O
    n_s = int(cb["sample"].split()[1])
    cores = os.cpu_count() or 1
    xs = []
    for li, a in enumerate(wl.acts):
        x = W.synth_activation(a, n_s, li, wl.dtype, "cpu")
        xs.append(x.view(torch.int16).numpy().view(np.uint16) if wl.dtype == "bf16" else x.numpy())

    def step():
        for li, (a, xh) in enumerate(zip(wl.acts, xs)):
            if wl.avg_bits is not None:
                mn, mx = O.group_minmax(xh)
                bits = O.allocate_bits(O.sensitivity(mn, mx), int(wl.avg_bits * n_s))
            else:
                bits = np.full(n_s, wl.bits, np.uint8)
            p, z, s, _ = O.quantize(xh, bits, W.quant_seed(li), 0, threads=cores)
            O.dequantize(p, z, s, bits, n_s, a.D, out_dtype=O.F32 if wl.dtype == "f32" else O.BF16,
                         threads=cores)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    s_in = 4 if wl.dtype == "f32" else 2
    E = n_s * sum(a.D for a in wl.acts)
    val = E * s_in / dt / 1e9
    cb = dict(cb, value=val)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": wl.dtype,
            "data": "synthetic (seeded ResNet-shaped activations, CPU generator)",
            "config": config_dict(wl, args, world, n_loc), "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ measurement
class Run:
    """One workload on this rank: inputs, the plan, the timed schedule."""

    def __init__(self, wl, n_loc, rank, world, dev, args, gather, torch, A, W, pool=0):
        from paper_2104_14129_b200.plan import ActivationSetPlan, PipelinedStep
        self.wl, self.n_loc, self.world = wl, n_loc, world
        self.s_in = 4 if wl.dtype == "f32" else 2
        tdt = torch.float32 if wl.dtype == "f32" else torch.bfloat16
        self.pool = pool
        if pool > 0:
            # per-layer streaming for sets larger than HBM (C5 below 4 GPUs): R
            # distinct resident buffers per tensor shape, the tensors of a shape
            # take them in turn (a forward pass writes each activation into
            # HBM just before it is compressed; the compressed set stays resident)
            bufs, occ = {}, {}
            self.xs = []
            for t, a in enumerate(wl.acts):
                key = (a.C, a.H, a.W, a.relu, a.image)
                k = occ.get(key, 0)
                occ[key] = k + 1
                lst = bufs.setdefault(key, [])
                if len(lst) < pool:
                    lst.append(W.synth_activation(a, n_loc, t + 100_000 * rank, wl.dtype, dev))
                self.xs.append(lst[k % pool])
            self.distinct_bytes = sum(x.numel() * x.element_size()
                                      for lst in bufs.values() for x in lst)
        else:
            self.xs = [W.synth_activation(a, n_loc, t + 100_000 * rank, wl.dtype, dev)
                       for t, a in enumerate(wl.acts)]
        torch.cuda.synchronize()
        self.plan = ActivationSetPlan(
            self.xs, [W.quant_seed(t) for t in range(len(wl.acts))], avg_bits=wl.avg_bits,
            bits=None if wl.avg_bits else wl.bits, n_total=n_loc * world,
            sample_base=rank * n_loc, gather=gather, meta=args.meta,
            level_mask=0x116 if args.levels == "pow2" else 0x1FE)
        max_numel = max(x.numel() for x in self.xs)
        # decompress streams (ACTNN_DQ_STREAMS, default 3), one output buffer each
        n_dq = max(1, int(os.environ.get("ACTNN_DQ_STREAMS", "3")))
        self.outs = [torch.empty(max_numel, dtype=tdt, device=dev) for _ in range(max(2, n_dq))]
        self.out_dt = A.api.F32 if wl.dtype == "f32" else A.api.BF16
        # the timed schedule (plan.PipelinedStep): statistics / quantisation
        # alternate over ACTNN_S_STREAMS / ACTNN_Q_STREAMS streams (default 2
        # each); allocation on a high-priority stream
        self.ps = PipelinedStep(self.plan, self.outs, self.out_dt, dev,
                                n_stats=int(os.environ.get("ACTNN_S_STREAMS", "2")),
                                n_quant=int(os.environ.get("ACTNN_Q_STREAMS", "2")), n_dq=n_dq)
        self.E_loc = n_loc * sum(a.D for a in wl.acts)
        self.graph_error = None

    def capture(self, dist_on, barrier):
        try:
            self.ps.capture(check_exchange=dist_on)
            barrier()
        except Exception as e:  # fall back to the eager schedule
            self.ps.graph = None
            self.graph_error = f"{type(e).__name__}: {e}"[:200]
            import torch
            torch.cuda.synchronize()
            barrier()

    def phases(self, torch, barrier, reps):
        """The schedule once more, eager, with events at the compress /
        decompress boundary (rank-local), averaged over `reps` steps."""
        ps = self.ps
        marks = []
        barrier()
        for _ in range(reps):
            m = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            m[0].record(ps.stream)
            ps.compress()
            m[1].record(ps.stream)
            ps.decompress()
            m[2].record(ps.stream)
            marks.append(m)
        barrier()
        t_comp = sum(m[0].elapsed_time(m[1]) for m in marks) / reps
        t_decomp = sum(m[1].elapsed_time(m[2]) for m in marks) / reps
        return t_comp, t_decomp

    def breakdown(self, torch, barrier, kb):
        """Serial per-kernel breakdown, two ways, both on the main stream with a
        spin kernel ahead of each pass (host enqueue gaps stay out of the events):
          - kernel-major sequence (the roofline's launch durations): K1 of every
            tensor back to back, then every [all-gather +] K2, every K3, every K4,
            one event pair around each kernel type's run of launches; a kernel's
            average launch duration = its run / the number of launches.  Each
            launch still runs alone (same stream, no overlap), ramp and tail
            included;
          - an event pair around every single launch (tensor-major order), which
            adds the per-event-pair overhead (~4-6 us measured on this part:
            tools/cuda_checks/small_write.cu times an empty kernel at 6 us) to
            every launch; kept as `per_launch_event_pairs` for comparison."""
        import ctypes
        plan, outs, out_dt = self.plan, self.outs, self.out_dt
        sp = ctypes.c_void_p(self.ps.stream.cuda_stream)
        nl = len(plan.layers)

        def events():
            per = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(nl)]
            per += [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(nl)]
            return per

        def serial(ev):
            for i in range(nl):
                plan.compress_layer(i, sp, ev[i])
            for i in range(nl):
                plan.decompress_layer(i, outs[i & 1], out_dt, sp, ev[nl + i])

        lib = plan.lib
        from paper_2104_14129_b200 import plan as plan_mod
        _lib_check, _ptr = plan_mod._lib.check, plan_mod._p

        def sequence(ev):
            ev[0].record()
            if plan.mixed:
                for L in plan.layers:
                    _lib_check(lib.actnn_group_stats(*L.args["stats"], sp))
            ev[1].record()
            if plan.mixed:
                for L in plan.layers:
                    if plan.gather is not None:
                        plan.gather(L.S, L.S_loc)
                    _lib_check(lib.actnn_allocate_bits(*L.args["alloc"], sp))
            ev[2].record()
            for L in plan.layers:
                _lib_check(plan.qfn(*L.args["quant"], sp))
            ev[3].record()
            for i, L in enumerate(plan.layers):
                _lib_check(plan.dfn(*L.args["dequant"], _ptr(outs[i & 1]), out_dt, sp))
            ev[4].record()

        with torch.cuda.stream(self.ps.stream):
            barrier()
            t_host = time.perf_counter()
            serial(events())
            t_host = time.perf_counter() - t_host
            barrier()
            evs = []
            for _ in range(kb):
                torch.cuda._sleep(int(1.5 * t_host * 2.0e9))
                ev = events()
                serial(ev)
                evs.append(ev)
            barrier()
            seqs = []
            for _ in range(kb):
                torch.cuda._sleep(int(1.5 * t_host * 2.0e9))
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                sequence(ev)
                seqs.append(ev)
            barrier()
        kseq = {"stats": 0.0, "quantize": 0.0, "dequantize": 0.0}
        for ev in seqs:
            if plan.mixed:
                kseq["stats"] += ev[0].elapsed_time(ev[1])
            kseq["quantize"] += ev[2].elapsed_time(ev[3])
            kseq["dequantize"] += ev[3].elapsed_time(ev[4])
        self.kt_seq = {k: v / kb for k, v in kseq.items()}
        # K2 (+ the exchange when k > 1) of every tensor back to back: latency-bound
        # single-CTA kernel, reported per launch (<= ~10 us)
        self.k2_seq_ms = (sum(ev[1].elapsed_time(ev[2]) for ev in seqs) / kb
                          if plan.mixed else None)
        kt = {"stats": 0.0, "quantize": 0.0, "dequantize": 0.0}
        tq = {"compress": 0.0, "decompress": 0.0}
        for per in evs:
            for i in range(nl):
                if plan.mixed:
                    kt["stats"] += per[i][0].elapsed_time(per[i][1])
                kt["quantize"] += per[i][2].elapsed_time(per[i][3])
                kt["dequantize"] += per[nl + i][0].elapsed_time(per[nl + i][1])
            tq["compress"] += per[0][0 if plan.mixed else 2].elapsed_time(per[nl - 1][3])
            tq["decompress"] += per[nl][0].elapsed_time(per[2 * nl - 1][1])
        self.layer_rows = None
        if os.environ.get("ACTNN_LAYER_DUMP"):
            self.layer_rows = [
                {"layer": i, "name": self.wl.acts[i].name, "N": L.N, "D": L.D,
                 "stats_us": 1e3 * sum(e[i][0].elapsed_time(e[i][1]) for e in evs) / kb
                 if plan.mixed else None,
                 "quant_us": 1e3 * sum(e[i][2].elapsed_time(e[i][3]) for e in evs) / kb,
                 "dequant_us": 1e3 * sum(e[nl + i][0].elapsed_time(e[nl + i][1])
                                         for e in evs) / kb}
                for i, L in enumerate(plan.layers)]
        return {k: v / kb for k, v in kt.items()}, {k: v / kb for k, v in tq.items()}

    def report(self, args, ms_step, t_comp, t_decomp, kt, tq, peak, peak_src):
        """The roofline / phase fields of a bench line for this workload."""
        plan, wl, world = self.plan, self.wl, self.world
        bits_host = plan.bits_host()
        alg = algorithmic_bytes(plan.layers, bits_host, self.s_in, self.s_in, plan.mixed,
                                4 if args.meta == "bf16" else 8)
        nl = len(plan.layers)
        # launch durations from the kernel-major sequence (breakdown docstring);
        # the per-launch event-pair numbers ride along for comparison
        kev = kt
        kt = getattr(self, "kt_seq", None) or kev
        dom = max(kt, key=lambda k: kt[k])
        ach = alg[dom] / (kt[dom] * 1e-3) / 1e9
        names = {"stats": "group_stats_kernel (K1)",
                 "quantize": "quantize_ws_kernel (K3)" if plan.mixed
                 else "quantize_fast_kernel (K3)",
                 "dequantize": "dequantize_fast_kernel (K4)"}
        roofline = {
            "bound": "hbm", "kernel": names[dom], "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak, "peak_source": peak_src,
            "frac_nominal": ach / NOMINAL_HBM_GBS, "peak_nominal": NOMINAL_HBM_GBS,
            "traffic": (ncu_traffic(dom, plan.mixed)
                        if wl.name == "c3" and args.meta == "f32" and args.levels == "pow2"
                        and self.pool == 0 else None),
            "algorithmic_bytes_per_launch": alg[dom] / nl,
            "avg_launch_us": kt[dom] * 1e3 / nl,
            "launch_timing": "kernel-major sequence: one event pair around the run of all "
                             f"{nl} launches of the kernel on its stream, each launch alone",
            "avg_launch_us_event_pairs": kev[dom] * 1e3 / nl,
            "launches_per_step": nl,
            # the same kernel inside the timed schedule: K4 is the only kernel of
            # the decompress phase (its launches overlap on several streams)
            "in_step": {"phase": f"decompress (K4 only, {len(self.ps.dq)} streams)",
                        "GBps": alg["dequantize"] / (t_decomp * 1e-3) / 1e9,
                        "frac": alg["dequantize"] / (t_decomp * 1e-3) / 1e9 / peak,
                        "frac_nominal": alg["dequantize"] / (t_decomp * 1e-3) / 1e9
                        / NOMINAL_HBM_GBS},
            "per_kernel": {k: {"kernel": names[k], "ms_per_step": kt[k],
                               "share_of_step": kt[k] / ms_step,
                               "GBps": (alg[k] / (kt[k] * 1e-3) / 1e9) if kt[k] else None,
                               "frac": (alg[k] / (kt[k] * 1e-3) / 1e9 / peak) if kt[k] else None,
                               "frac_nominal": (alg[k] / (kt[k] * 1e-3) / 1e9 / NOMINAL_HBM_GBS)
                               if kt[k] else None,
                               "algorithmic_bytes_per_step": alg[k],
                               "ms_per_step_event_pairs": kev[k],
                               "frac_event_pairs": (alg[k] / (kev[k] * 1e-3) / 1e9 / peak)
                               if kev[k] else None}
                           for k in kt}}
        k2 = getattr(self, "k2_seq_ms", None)
        if k2:
            roofline["per_kernel"]["allocate"] = {
                "kernel": "allocate_kernel (K2)" + (" + all-gather of S" if plan.gather else ""),
                "bound": "latency (one CTA; overlapped with K1 / K3 of other tensors in the step)",
                "ms_per_step": k2, "us_per_launch": k2 * 1e3 / nl,
                "samples_per_launch": plan.layers[0].S.numel()}
        total_alg = sum(alg.values())
        avg_bits = [float(b.double().mean()) for b in bits_host]
        E = world * self.E_loc * self.s_in
        return {
            "compress_GBps": E / (t_comp * 1e-3) / 1e9,
            "decompress_GBps": E / (t_decomp * 1e-3) / 1e9,
            "compress_ms": t_comp, "decompress_ms": t_decomp,
            "compress_frac": (alg["stats"] + alg["quantize"]) / (t_comp * 1e-3) / 1e9 / peak,
            "decompress_frac": alg["dequantize"] / (t_decomp * 1e-3) / 1e9 / peak,
            "serial_breakdown_ms": {"compress": tq["compress"], "decompress": tq["decompress"]},
            "hbm_frac_step": total_alg / (ms_step * 1e-3) / 1e9 / peak,
            "hbm_frac_step_nominal": total_alg / (ms_step * 1e-3) / 1e9 / NOMINAL_HBM_GBS,
            "algorithmic_bytes_per_step": total_alg,
            "roofline": roofline,
            "avg_bits_realised": sum(avg_bits) / len(avg_bits),
        }


def time_steps(ps, steps, barrier, torch, clk=None):
    """K steps between one event pair, barrier + synchronize on both sides."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(ps.stream)
    for _ in range(steps):
        ps()
    e1.record(ps.stream)
    barrier()
    return e0.elapsed_time(e1)


def run_side(name, args, dev, torch, A, W, peak, peak_src, barrier):
    """A side leg (N = 1, outside the headline timed region): the C2 / C4
    workload through the same schedule, graph-replayed, with its own phase
    split, roofline and per-kernel breakdown, so that the driver's record holds
    all three single-GPU configs."""
    wl = W.workload(name)
    r = Run(wl, wl.N, 0, 1, dev, args, None, torch, A, W)
    with torch.cuda.stream(r.ps.stream):
        for _ in range(3):
            r.ps()
    barrier()
    r.capture(False, barrier)
    ms = time_steps(r.ps, args.side_steps, barrier, torch) / args.side_steps
    t_comp, t_decomp = r.phases(torch, barrier, min(args.side_steps, 5))
    kt, tq = r.breakdown(torch, barrier, 3)
    rep = r.report(args, ms, t_comp, t_decomp, kt, tq, peak, peak_src)
    out = {"workload": f"{wl.name.upper()}: {wl.description}", "dtype": wl.dtype,
           "value": r.E_loc * r.s_in / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
           "steps": args.side_steps, "cuda_graph": r.ps.graph is not None,
           "gpu_launches_per_step": r.plan.launches_per_step()}
    out.update(rep)
    del r
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def oracle_minmax_threaded(O, xh, threads):
    """O3 over sample slices on `threads` host threads (ctypes drops the GIL)."""
    import numpy as np
    N = xh.shape[0]
    k = max(1, min(threads, N))
    bounds = [(N * i // k, N * (i + 1) // k) for i in range(k)]
    parts = [None] * k

    def go(i):
        parts[i] = O.group_minmax(xh[bounds[i][0]:bounds[i][1]])

    ts = [threading.Thread(target=go, args=(i,)) for i in range(k)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


def oracle_phases(wl, torch, threads, target_s):
    """The oracle, as it stands, on a bounded sample of the workload (the first
    n_s samples of every tensor), each phase timed: stats + allocation (O3,
    O11, O12), quantise + pack (O4-O9), unpack + dequantise (O10).  n_s is
    calibrated so the run takes ~target_s.  Returns per-phase elements/s."""
    import numpy as np
    import oracle as O
    from paper_2104_14129_b200 import workloads as W
    acts = wl.acts

    def inputs(n):
        out = []
        for li, a in enumerate(acts):
            x = W.synth_activation(a, n, li, wl.dtype, "cpu")
            out.append(x.view(torch.int16).numpy().view(np.uint16) if wl.dtype == "bf16"
                       else x.numpy())
        return out

    def run(n_s, xs):
        t = {"stats_alloc": 0.0, "quantize_pack": 0.0, "unpack_dequantize": 0.0}
        for li, (a, xh) in enumerate(zip(acts, xs)):
            t0 = time.perf_counter()
            if wl.avg_bits is not None:
                mn, mx = oracle_minmax_threaded(O, xh, threads)
                bits = O.allocate_bits(O.sensitivity(mn, mx), int(wl.avg_bits * n_s))
            else:
                bits = np.full(n_s, wl.bits, np.uint8)
            t1 = time.perf_counter()
            packed, zmin, scale, _ = O.quantize(xh, bits, W.quant_seed(li), 0, threads=threads)
            t2 = time.perf_counter()
            O.dequantize(packed, zmin, scale, bits, n_s, a.D,
                         out_dtype=O.F32 if wl.dtype == "f32" else O.BF16, threads=threads)
            t3 = time.perf_counter()
            t["stats_alloc"] += t1 - t0
            t["quantize_pack"] += t2 - t1
            t["unpack_dequantize"] += t3 - t2
        return t

    n_s = 1
    while True:
        xs = inputs(n_s)
        t = run(n_s, xs)
        tot = sum(t.values())
        if tot >= target_s / 4 or n_s >= wl.N:
            break
        n_s = min(wl.N, 2 * n_s)
    n_new = max(1, min(wl.N, int(n_s * target_s / max(tot, 1e-3))))
    if n_new > n_s:
        n_s = n_new
        xs = inputs(n_s)
        t = run(n_s, xs)
    E = n_s * sum(a.D for a in acts)
    s_in = 4 if wl.dtype == "f32" else 2
    tot = sum(t.values())
    return {"threads": threads, "samples_per_tensor": n_s, "elements": E, "seconds": tot,
            "GBps_in": E * s_in / tot / 1e9, "elements_per_s": E / tot,
            "phases_elements_per_s": {k: (E / v if v > 0 else None) for k, v in t.items()},
            "phases_seconds": t}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------------ main arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return 0

    import torch
    import torch.distributed as dist

    import paper_2104_14129_b200 as A
    from paper_2104_14129_b200 import dist as AD
    from paper_2104_14129_b200 import workloads as W

    # one process per GPU; ACTNN_DIST_BACKEND=gloo is a test mode in which
    # several ranks may share a GPU (NCCL refuses duplicate devices)
    backend = os.environ.get("ACTNN_DIST_BACKEND", "nccl")
    # ACTNN_FORCE_DIST=1: the multi-rank code path (process group, all-gather of
    # S, graph capture of the collectives) even at world size 1 -- a test mode
    dist_on = world > 1 or os.environ.get("ACTNN_FORCE_DIST") == "1"
    if dist_on:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", str(world))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if dist_on:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def barrier():
        if dist_on:
            dist.barrier(device_ids=[local]) if backend == "nccl" else dist.barrier()
        torch.cuda.synchronize()

    wl = W.workload(args.config)
    n_loc = wl.N // world if args.config == "c5" else wl.N
    s_in = 4 if wl.dtype == "f32" else 2
    # C5 (batch 4096, 365.8 GB of bf16 activations) is resident from 4 GPUs on;
    # below that its tensors are streamed through a pool of per-shape buffers
    need = n_loc * sum(a.D for a in wl.acts) * s_in * 1.15
    free = torch.cuda.mem_get_info(dev)[0]
    pool = args.pool
    if pool == 0 and need > free:
        pool = 2
    gather = AD.make_gather(world, backend) if dist_on else None
    run = Run(wl, n_loc, rank, world, dev, args, gather, torch, A, W, pool=pool)
    ps = run.ps
    torch.cuda.set_stream(ps.stream)
    plan = run.plan

    for _ in range(max(3, args.warmup)):
        ps()
    barrier()
    # capture the whole pipelined step in one CUDA graph (removes the ~430
    # per-step CPU launches; every kernel still runs on every replay).  N > 1:
    # the NCCL all-gathers are captured too (tests check replay == eager);
    # ACTNN_DIST_GRAPH=0 keeps the multi-GPU step eager
    if args.graph is None:
        args.graph = not dist_on or (backend == "nccl"
                                    and os.environ.get("ACTNN_DIST_GRAPH", "1") != "0")
    if args.graph:
        run.capture(dist_on, barrier)
        args.graph = ps.graph is not None

    # ---- headline: K steps, one event pair, max over ranks
    with ClockSampler(local) as clk:
        ms = time_steps(ps, args.steps, barrier, torch)
    if dist_on:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = world * run.E_loc * s_in / (ms_step * 1e-3) / 1e9

    t_comp, t_decomp = run.phases(torch, barrier, min(args.steps, 5))
    kt, tq = run.breakdown(torch, barrier, max(3, args.steps // 4))
    if run.layer_rows is not None and rank == 0:
        with open(os.environ["ACTNN_LAYER_DUMP"], "w") as f:
            json.dump(run.layer_rows, f, indent=0)
    peak, peak_src = hbm_peak()
    rep = run.report(args, ms_step, t_comp, t_decomp, kt, tq, peak, peak_src)
    xs = run.xs

    # ---- NEXT-3 / NEXT-4 side measurements (not part of the step)
    adapt = None
    if plan.mixed and world == 1 and not args.no_adapt and pool == 0:
        adapt = run_adapt(A, plan, xs, wl, s_in, torch, peak, barrier)
    contexts = None
    if world == 1 and not args.no_adapt:
        contexts = run_contexts(A, xs, wl, torch, peak, barrier)
    # ---- e2e through the public API with host buffers (per-layer pipeline)
    e2e = None
    if not args.no_e2e:
        import ctypes
        e2e = run_e2e(args, plan, xs, run.outs, run.out_dt, ctypes.c_void_p(ps.stream.cuda_stream),
                      ps.stream, world, local, dev, torch, dist, s_in, run.E_loc, barrier,
                      backend, unique_inputs=(pool == 0))

    cfg = dict(config_dict(wl, args, world, n_loc),
               **({"graph_error": run.graph_error} if run.graph_error else {}))
    if pool:
        cfg["inputs"] = (f"streamed per layer: {pool} distinct resident buffers per tensor "
                         f"shape ({run.distinct_bytes / 1e9:.1f} GB), reused by that shape's "
                         f"tensors; the whole set ({need / 1.15 / 1e9:.1f} GB per GPU) exceeds "
                         "HBM. The compressed set of every tensor stays resident.")
        cfg["l2"] = "every tensor >= 16 MB, consecutive tensors use distinct buffers"
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if args.config != "c5" else "strong",
            "vs_baseline": None, "dtype": wl.dtype,
            "data": "synthetic (seeded ResNet-shaped activations generated on the GPU)",
            "config": cfg}
    line.update(rep)
    line.update({"gpu_launches": plan.launches_per_step() * args.steps,
                 "clocks": clk.summary(),
                 "paper_context": PAPER_CONTEXT})
    if e2e is not None:
        line["e2e"] = e2e
    if adapt is not None:
        line["adapt"] = adapt
    if contexts is not None:
        line["contexts"] = contexts
    if world == 1 and plan.mixed and not args.no_adapt:
        line["allocator_latency"] = run_k2_latency(A, max(L.D for L in plan.layers), dev, torch)
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        allc = oracle_phases(wl, torch, cores, args.cpu_seconds * 0.6)
        one = oracle_phases(wl, torch, 1, args.cpu_seconds * 0.4)
        line["cpu_baseline"] = {
            "value": allc["GBps_in"], "unit": "GB/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"first {allc['samples_per_tensor']} of {wl.N} samples of each of the "
                      f"{len(wl.acts)} tensors ({allc['elements']} elements), full compress + "
                      f"decompress (stats, heap allocation, quantize, dequantize) on all "
                      f"{cores} host threads, {allc['seconds']:.1f} s",
            "all_cores": allc, "single_thread": one}
    # ---- side legs: the other single-GPU configs of BASELINE.json (C2, C4)
    if world == 1 and args.config == "c3" and not args.no_side:
        del xs, adapt, contexts
        free_run(run, torch)
        del run, ps, plan
        torch.cuda.set_stream(torch.cuda.default_stream())
        torch.cuda.empty_cache()
        line["side"] = {}
        for name in ("c2", "c4"):
            try:
                line["side"][name] = run_side(name, args, dev, torch, A, W, peak, peak_src,
                                              barrier)
            except Exception as e:  # a side leg never voids the headline line
                line["side"][name] = {"error": f"{type(e).__name__}: {e}"[:300]}
                torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()
    return 0


def free_run(run, torch):
    run.ps.graph = None
    run.plan.layers.clear()
    run.xs.clear()
    run.outs.clear()
    torch.cuda.synchronize()


def run_contexts(A, xs, wl, torch, peak, barrier, reps=5):
    """NEXT-4 side measurement: the lossless contexts of a Conv-BN-ReLU-MaxPool
    block on the largest tensor of the set (ResNet stem, 64 x 112 x 112 per
    sample): ReLU 1-bit mask pack (+ y) and its backward, 3x3/2 max pool with
    the 8-bit argmax and its backward.  Algorithmic bytes per call / event time."""
    x = max(xs, key=lambda t: t.numel())
    N = x.shape[0]
    C, H, W = 64, 112, 112
    if x.numel() != N * C * H * W:
        return None
    x4 = x.view(N, C, H, W)
    s = x.element_size()
    E = x.numel()
    cs = torch.cuda.current_stream()

    def t(fn):
        fn()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        for _ in range(reps):
            fn()
        b.record(cs)
        b.synchronize()
        return a.elapsed_time(b) / reps

    mask, y = A.relu_pack(x, want_y=True)
    t_pack = t(lambda: A.relu_pack(x, want_y=True))
    t_rb = t(lambda: A.relu_backward(mask, x))
    yp, idx = A.maxpool2d(x4, 3, 2, 1)
    t_pf = t(lambda: A.maxpool2d(x4, 3, 2, 1))
    t_pb = t(lambda: A.maxpool2d_backward(idx, yp, H, W, 3, 2, 1))
    EO = yp.numel()
    rows = {"relu_pack": (t_pack, E * s + E // 8 + E * s),
            "relu_backward": (t_rb, E // 8 + 2 * E * s),
            "maxpool2d_forward": (t_pf, E * s + EO * (s + 1)),
            "maxpool2d_backward": (t_pb, EO * (s + 1) + E * s)}
    return {k: {"ms": ms, "GBps": by / (ms * 1e-3) / 1e9, "frac": by / (ms * 1e-3) / 1e9 / peak,
                "algorithmic_bytes": by} for k, (ms, by) in rows.items()} | {
        "tensor": f"{N}x{C}x{H}x{W} {wl.dtype}", "note": "NEXT-4 (P:1388-1419) side measurement, "
        "not part of the step"}


def run_adapt(A, plan, xs, wl, s_in, torch, peak, barrier, reps=5):
    """K6 over every tensor (event pair per launch) and K5 on the [L, N]
    sensitivities of this step, timed on the current stream."""
    outs = [torch.empty(x.shape[0], dtype=torch.float64, device=x.device) for x in xs]
    ws = [torch.zeros(int(A._lib.load().actnn_workspace_bytes(2, x.shape[0],
                                                             x.numel() // x.shape[0], 256)) + 8,
                      dtype=torch.uint8, device=x.device) for x in xs]
    lib = A._lib.load()
    cs = torch.cuda.current_stream()
    sp = __import__("ctypes").c_void_p(cs.cuda_stream)

    def sqnorm(i):
        x = xs[i]
        N = x.shape[0]
        A._lib.check(lib.actnn_grad_sqnorm(A.api._ptr(x), A.api._dtype_code(x.dtype), N,
                                           x.numel() // N, 256, A.api._ptr(outs[i]),
                                           A.api._ptr(ws[i]), ws[i].numel(), sp))

    for i in range(len(xs)):
        sqnorm(i)
    barrier()
    t_k6 = 0.0
    for _ in range(reps):
        for i in range(len(xs)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cs)
            sqnorm(i)
            b.record(cs)
            b.synchronize()
            t_k6 += a.elapsed_time(b)
    t_k6 /= reps
    # kernel-major sequence (as the roofline's launch durations): one event pair
    # around the run of all launches, each launch alone on the stream
    t_seq = 0.0
    for _ in range(reps):
        torch.cuda._sleep(20_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        for i in range(len(xs)):
            sqnorm(i)
        b.record(cs)
        b.synchronize()
        t_seq += a.elapsed_time(b) / reps
    nbytes = sum(x.numel() for x in xs) * s_in
    D = [L.D for L in plan.layers]
    N = plan.layers[0].N
    sens = torch.stack([L.S[:N] for L in plan.layers]).contiguous()
    gscale = torch.stack(outs).contiguous()  # ||grad_n||^2 estimates of this step
    alloc = A.LayerAllocator(D, N, xs[0].device, plan.level_mask)
    b_total = int(wl.avg_bits * N * sum(D))
    alloc(sens, b_total, gscale)
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cs)
    for _ in range(reps):
        bits, budgets = alloc(sens, b_total, gscale)
    b.record(cs)
    b.synchronize()
    t_k5 = a.elapsed_time(b) / reps
    used = int((budgets.cpu() * torch.tensor(D)).sum())
    return {"grad_sqnorm": {"kernel": "grad_sqnorm_kernel (K6)", "ms_per_set": t_seq,
                            "GBps": nbytes / (t_seq * 1e-3) / 1e9,
                            "frac": nbytes / (t_seq * 1e-3) / 1e9 / peak,
                            "launch_timing": "kernel-major sequence (mean of reps)",
                            "ms_per_set_event_pairs": t_k6,
                            "frac_event_pairs": nbytes / (t_k6 * 1e-3) / 1e9 / peak,
                            "launches": len(xs)},
            "stage2": {"kernel": "allocate_layers_kernel (K5)", "us": t_k5 * 1e3,
                       "layers": len(D), "samples": N,
                       "moves": len(D) * N * (bin(plan.level_mask).count("1") - 1),
                       "b_total": b_total, "bits_used": used},
            "note": "NEXT-3 (P:553-569) side measurement, not part of the step; the "
                    "activations stand in for same-shaped gradients"}


def run_k2_latency(A, D, dev, torch, reps=50):
    """K2 (actnn_allocate_bits) alone at batch sizes N = 256 .. 16384 on seeded
    log-normal sensitivities (avg 2 bits over {1, 2, 4, 8}): per-launch time of
    `reps` back-to-back launches, and one launch after an idle gap (event pair
    included).  SURVEY §6 item 5 wants <= ~10 us at N = 4096."""
    out = {}
    cs = torch.cuda.current_stream()
    g = torch.Generator(device="cpu").manual_seed(20260)
    for N in (256, 1024, 4096, 16384):
        S = torch.exp(2.0 * torch.randn(N, generator=g, dtype=torch.float64)).to(dev)
        budget = 2 * N
        A.allocate_bits(S, budget, D)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record(cs)
        for _ in range(reps):
            A.allocate_bits(S, budget, D)
        b.record(cs)
        b.synchronize()
        seq = a.elapsed_time(b) / reps
        one = 1e9
        for _ in range(5):
            torch.cuda._sleep(2_000_000)
            a.record(cs)
            A.allocate_bits(S, budget, D)
            b.record(cs)
            b.synchronize()
            one = min(one, a.elapsed_time(b))
        out[str(N)] = {"us_back_to_back": round(seq * 1e3, 2), "us_single": round(one * 1e3, 2)}
    return {"kernel": "allocate_kernel (K2)", "D": D, "levels": "{1,2,4,8}", "avg_bits": 2,
            "by_N": out,
            "note": "us_back_to_back includes the allocation of the (bits, off) outputs by the "
                    "Python wrapper (caching allocator); us_single includes one event pair"}


def run_e2e(args, plan, xs, outs, out_dt, sp, stream, world, local, dev, torch, dist, s_in,
            E_loc, barrier, backend="nccl", unique_inputs=True):
    """Host-pinned inputs copied in, compressed, decompressed and copied back
    out every step (per-tensor pipeline over three streams)."""
    import psutil
    in_bytes = sum(x.numel() * x.element_size() for x in xs)
    max_b = max(x.numel() * x.element_size() for x in xs)
    if psutil.virtual_memory().available < (in_bytes + 3 * max_b) * 1.2 * world:
        return {"value": None, "unit": "GB/s", "skipped": "not enough host memory for pinned "
                "inputs", "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": in_bytes}
    host_in = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in xs]
    for h, x in zip(host_in, xs):
        h.copy_(x)
    host_out = [torch.empty(outs[0].numel(), dtype=outs[0].dtype, pin_memory=True)
                for _ in range(3)]
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    nl = len(xs)
    sample = max(1, int(os.environ.get("ACTNN_E2E_STEPS", args.e2e_steps)))

    def e2e_step():
        ev_in = [torch.cuda.Event() for _ in range(nl)]
        ev_dq = [torch.cuda.Event() for _ in range(nl)]
        ev_out = [torch.cuda.Event() for _ in range(nl)]
        with torch.cuda.stream(h2d):
            for i in range(nl):
                xs[i].copy_(host_in[i], non_blocking=True)
                ev_in[i].record(h2d)
        for i in range(nl):
            stream.wait_event(ev_in[i])
            if i >= 2:
                stream.wait_event(ev_out[i - 2])   # device out slot i&1 drained
            plan.compress_layer(i, sp)
            plan.decompress_layer(i, outs[i & 1], out_dt, sp)
            ev_dq[i].record(stream)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_dq[i])
                n = xs[i].numel()
                host_out[i % 3][:n].copy_(outs[i & 1][:n], non_blocking=True)
                ev_out[i].record(d2h)
        stream.wait_stream(d2h)
        stream.wait_stream(h2d)

    e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(sample):
        e2e_step()
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1) / sample
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64,
                          device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return {"value": world * E_loc * s_in / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "ms_per_step": ms, "steps": sample,
            "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": in_bytes,
            "path": "pinned host -> H2D -> actnn_group_stats/allocate/quantize/dequantize "
                    "(C ABI via plan) -> D2H pinned host, per-tensor pipelined on 3 streams"}


if __name__ == "__main__":
    sys.exit(main())
