for rep in 1 2; do for v in default pdl0; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  timeout 600 python tools/with_variant.py $L -- bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-adapt --no-side > gpurun_out/r02_b34_$v.log 2>&1
  echo "$v $(python tools/bl.py gpurun_out/r02_b34_$v.log)"
done; done
