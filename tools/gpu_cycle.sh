#!/bin/bash
# One GPU iteration: smoke, parity tests, short bench, ncu --set full on one layer.
# Usage (under gpurun): bash tools/gpu_cycle.sh TAG [LAYERS]
TAG=${1:-x}; LAYERS=${2:-1}
python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.log").read().strip().splitlines()[-1]); r = d["roofline"]
print("value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), {k: (round(v["ms_per_step"], 3), round(v["frac"], 3)) for k, v in r["per_kernel"].items()})
PY
if [ "$LAYERS" != "none" ]; then
timeout 800 ncu --set full --clock-control none --import-source on -k regex:"^quantize_|^dequantize_fast|^group_stats|^allocate" -s 4 -c 4 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 1 --layers $LAYERS > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
fi
