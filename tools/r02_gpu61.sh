#!/bin/bash
# Single pass through the warp-specialised K3 (producers take the statistics from the
# staged tile): GPU suite with it for fp32 and bf16 (wst2), C2 timings.
V=paper_2104_14129_b200/csrc/build
timeout 1500 python tools/with_variant.py $V/var_wst2/libactnn.so -- -m pytest tests -m gpu -q -x > gpurun_out/s61_pytest_wst2.log 2>&1; echo pytest_wst2=$?; tail -1 gpurun_out/s61_pytest_wst2.log
for rep in 1 2; do for v in default wst1 wst1s2; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=$V/var_$v/libactnn.so
  timeout 600 python tools/with_variant.py $L -- bench.py --config c2 --no-cpu --no-e2e --no-adapt > gpurun_out/s61_${v}_$rep.log 2>&1
  echo "$v $rep $(python tools/bl.py gpurun_out/s61_${v}_$rep.log)"
done; done
