# K3 with room for a co-resident K1 CTA (12 + 3 warps; 8 + 2 warps capped at 1 CTA/SM) vs 16 + 4: C4 and C3 steps
for rep in 1 2; do for v in default ws12 ws8; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  timeout 600 python tools/with_variant.py $L -- bench.py --config c4 --steps 5 --warmup 3 --no-cpu --no-e2e --no-adapt --no-side > gpurun_out/r02_b40_c4_$v.log 2>&1
  echo "c4 $v $(python tools/bl.py gpurun_out/r02_b40_c4_$v.log)"
  timeout 600 python tools/with_variant.py $L -- bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-adapt --no-side > gpurun_out/r02_b40_c3_$v.log 2>&1
  echo "c3 $v $(python tools/bl.py gpurun_out/r02_b40_c3_$v.log)"
done; done
for v in default dqu8 dqs6; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "c4 $v $(PROBE_CONFIG=c4 PROBE_SIZES=1 timeout 600 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1)"
done
