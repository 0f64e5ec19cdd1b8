#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adapt.py -q -x -k "allocate or mixed or virtual or stage" > gpurun_out/s66_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/s66_pytest.log
timeout 300 python tools/k2_latency.py | cut -c80-400
python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_k2prof/libactnn.so -- tools/k2_phases.py
