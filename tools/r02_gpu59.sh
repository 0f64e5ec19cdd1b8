#!/bin/bash
# C4 step with the bf16 K3 grid leaving k SMs to the next tensor's K1 (SM partitioning).
for rep in 1 2; do for v in default lv8 lv16 lv28 lv40; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  timeout 600 python tools/with_variant.py $L -- bench.py --config c4 --steps 5 --no-cpu --no-e2e --no-adapt > gpurun_out/s59_${v}_$rep.log 2>&1
  echo "$v $rep $(python tools/bl.py gpurun_out/s59_${v}_$rep.log)"
done; done
