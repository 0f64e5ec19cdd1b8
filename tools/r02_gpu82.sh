#!/bin/bash
# K2 with device asserts on every shared-memory index (compute-sanitizer is closed on the
# pool): the allocation, mixed-path, virtual-rank, stage-2 and C3/C5 whole-path tests.
V=paper_2104_14129_b200/csrc/build/var_k2assert/libactnn.so
timeout 1500 python tools/with_variant.py $V -- -m pytest tests/test_gpu_parity.py tests/test_gpu_full_parity.py tests/test_gpu_adapt.py tests/test_gpu_bf16meta.py -q -x -k "allocate or mixed or virtual or stage or c3_whole or c5 or n4096 or bf16meta" 2>&1 | tail -3
timeout 300 python tools/with_variant.py $V -- tools/k2_latency.py | cut -c80-330
