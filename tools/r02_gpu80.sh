#!/bin/bash
# K1 through a TMA ring (default, 3 stages) vs the LDG kernel (k1ldg) vs 2 / 4 stages.
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_parity.py tests/test_gpu_bf16meta.py -q -x -k "stats or mixed or c3 or c4 or virtual or bf16meta or c5" > gpurun_out/s80_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/s80_pytest.log
V=paper_2104_14129_b200/csrc/build
for rep in 1 2; do for v in default k1ldg k1s2 k1s4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=$V/var_$v/libactnn.so
  timeout 900 python tools/with_variant.py $L -- bench.py --no-cpu --no-e2e --no-adapt --no-side > gpurun_out/s80_c3_${v}_$rep.log 2>&1
  echo "c3 $v $rep $(python tools/bl.py gpurun_out/s80_c3_${v}_$rep.log)"
done; done
for v in default k1ldg; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=$V/var_$v/libactnn.so
  timeout 900 python tools/with_variant.py $L -- bench.py --config c4 --steps 5 --no-cpu --no-e2e --no-adapt > gpurun_out/s80_c4_${v}.log 2>&1
  echo "c4 $v $(python tools/bl.py gpurun_out/s80_c4_${v}.log)"
done
