#!/bin/bash
# Under gpurun: parity of the quantiser paths, C3 + C4 short benches, and an
# ncu --set full capture of the C4 layer-1 kernels.  Usage: bash tools/k3_cycle.sh TAG
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_$TAG.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_$TAG.log 2>&1; echo c4=$?
python tools/bl.py gpurun_out/bench_c3_$TAG.log gpurun_out/bench_c4_$TAG.log
if [ "${NCU:-1}" = "1" ]; then
timeout 800 ncu --set full --clock-control none --import-source on -k regex:"^quantize_|^group_stats" -s 3 -c 2 -o gpurun_out/prof_$TAG python tools/profile_step.py --config c4 --steps 1 --layers 1 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
fi
