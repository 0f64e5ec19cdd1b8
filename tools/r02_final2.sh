#!/bin/bash
# Round-2 closing evidence on the final code: smoke, GPU suite, default bench line,
# ncu launch list + --set full captures (tools/make_profiles.sh r02).
T=r02g
python __graft_entry__.py > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c3.log 2>&1; echo c3=$?
python tools/bl.py gpurun_out/${T}_bench_c3.log
bash tools/make_profiles.sh r02
