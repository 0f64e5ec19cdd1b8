#!/bin/bash
V=paper_2104_14129_b200/csrc/build
timeout 900 python tools/with_variant.py $V/var_k2t1k/libactnn.so -- -m pytest tests/test_gpu_parity.py -q -x -k "allocate" 2>&1 | tail -1
echo "512: $(timeout 300 python tools/k2_latency.py | cut -c80-330)"
echo "1024: $(timeout 300 python tools/with_variant.py $V/var_k2t1k/libactnn.so -- tools/k2_latency.py | cut -c80-330)"
python tools/with_variant.py $V/var_k2t1kprof/libactnn.so -- tools/k2_phases.py
