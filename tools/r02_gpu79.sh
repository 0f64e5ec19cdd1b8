#!/bin/bash
for rep in 1 2; do for v in default notab4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  timeout 900 python tools/with_variant.py $L -- bench.py --config c4 --steps 5 --no-cpu --no-e2e --no-adapt > gpurun_out/s79_${v}_$rep.log 2>&1
  echo "$v $rep $(python tools/bl.py gpurun_out/s79_${v}_$rep.log)"
done; done
