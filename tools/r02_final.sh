#!/bin/bash
# Round-2 final evidence (after the K2 change): smoke, GPU suite, bench lines (C3 default
# with side legs, reference arm), ncu launch list + --set full captures, sanitizers on K2.
T=r02f
python __graft_entry__.py > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.log 2>&1; echo ref=$?
python tools/bl.py gpurun_out/${T}_bench_c3.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck initcheck synccheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "allocate" > gpurun_out/${T}_sanitize_k2_$tool.log 2>&1
  echo "k2 $tool rc=$? $(tail -1 gpurun_out/${T}_sanitize_k2_$tool.log) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${T}_sanitize_k2_$tool.log | tail -1)"
done
bash tools/make_profiles.sh r02
