#!/bin/bash
# Re-entry check after the container re-creation: smoke, GPU suite, default bench line.
python __graft_entry__.py > gpurun_out/s47_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s47_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/s47_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/s47_bench_c3.log 2>&1; echo c3=$?
tail -1 gpurun_out/s47_bench_c3.log | cut -c1-600
