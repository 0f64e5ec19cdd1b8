#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s70_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/s70_pytest_gpu.log
timeout 300 python tools/k2_latency.py | cut -c80-330
