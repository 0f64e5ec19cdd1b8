#!/bin/bash
# K2 with the keys staged in shared memory (32-bit loop indices): parity + latency + ncu.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adapt.py -q -x -k "allocate or mixed or virtual or stage" > gpurun_out/s53_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/s53_pytest.log
timeout 300 python tools/k2_latency.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"allocate_kernel" -s 2 -c 1 \
  -o gpurun_out/r02_k2b_4096 python tools/k2_once.py 4096 > gpurun_out/s53_ncu.log 2>&1; echo ncu=$?
