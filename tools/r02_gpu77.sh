#!/bin/bash
# bf16-output K4 at b <= 2 through byte-permute table selects: GPU suite, C4 K4 per size.
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s77_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/s77_pytest.log
for v in default notab; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "c4 $v $(PROBE_CONFIG=c4 PROBE_SIZES=1 timeout 900 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -2 | tr '\n' ' ')"
done
