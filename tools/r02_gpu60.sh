#!/bin/bash
# K2 histogram variants: 0 two 32-bit histograms + match.any, 1 (default) packed 64-bit +
# match.any, 2 packed 64-bit per lane.
for v in default k2h0 k2h2; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v $(timeout 300 python tools/with_variant.py $L -- tools/k2_latency.py | cut -c80-400)"
  timeout 900 python tools/with_variant.py $L -- -m pytest tests/test_gpu_parity.py -q -x -k "allocate" 2>&1 | tail -1
done
python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_k2prof/libactnn.so -- tools/k2_phases.py
