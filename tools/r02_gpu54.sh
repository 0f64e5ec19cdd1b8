#!/bin/bash
V=paper_2104_14129_b200/csrc/build/var_k2t1024/libactnn.so
echo "512: $(timeout 300 python tools/k2_latency.py)"
echo "1024: $(timeout 300 python tools/with_variant.py $V -- tools/k2_latency.py)"
timeout 900 python tools/with_variant.py $V -- -m pytest tests/test_gpu_parity.py -q -x -k "allocate" 2>&1 | tail -1
