#!/bin/bash
# Under gpurun: the round's evidence -- smoke, GPU parity suite, one bench line per
# config (C3 default with e2e + CPU baseline; C2; C4; C3 with bf16 metadata; C3 with
# the unit-step allocator), then the ncu captures of tools/make_profiles.sh.
TAG=${1:-r01}
python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c2 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c2.log 2>&1; echo c2=$?
timeout 900 python bench.py --config c4 --steps 5 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --meta bf16 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c3_bf16meta.log 2>&1; echo bf16meta=$?
timeout 600 python bench.py --levels unit --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c3_unit.log 2>&1; echo unit=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.log 2>&1; echo ref=$?
python tools/bl.py gpurun_out/${TAG}_bench_*.log
if [ "${PROFILES:-1}" = "1" ]; then bash tools/make_profiles.sh ${TAG}; fi
