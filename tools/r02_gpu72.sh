#!/bin/bash
V=paper_2104_14129_b200/csrc/build
for rep in 1 2; do for v in default sp13; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=$V/var_$v/libactnn.so
  timeout 600 python tools/with_variant.py $L -- bench.py --config c2 --no-cpu --no-e2e --no-adapt > gpurun_out/s72_${v}_$rep.log 2>&1
  echo "$v $rep $(python tools/bl.py gpurun_out/s72_${v}_$rep.log)"
done; done
