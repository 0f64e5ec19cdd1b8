#!/bin/bash
# bf16-output K4: table selects with 3 stages (default) vs the round-2 kernel (no table, 4
# stages) vs no table with 3 stages; C4 per size class.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16meta.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in default notab4 notab3; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "c4 $v $(PROBE_CONFIG=c4 PROBE_SIZES=1 timeout 900 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-700)"
done; done
