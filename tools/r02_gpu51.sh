#!/bin/bash
# K2 with the sample weights staged in shared memory: parity + latency.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "allocate or mixed or virtual" > gpurun_out/s51_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/s51_pytest.log
timeout 300 python tools/k2_latency.py
