#!/bin/bash
V=paper_2104_14129_b200/csrc/build
timeout 900 python tools/with_variant.py $V/var_k2nm/libactnn.so -- -m pytest tests/test_gpu_parity.py -q -x -k "allocate" 2>&1 | tail -1
timeout 300 python tools/with_variant.py $V/var_k2nm/libactnn.so -- tools/k2_latency.py | cut -c80-400
python tools/with_variant.py $V/var_k2nmprof/libactnn.so -- tools/k2_phases.py
