#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adapt.py -q -x -k "allocate or mixed or virtual or stage" > gpurun_out/s56_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/s56_pytest.log
timeout 300 python tools/k2_latency.py
