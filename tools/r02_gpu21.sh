# C2 single pass: straight-line full-unit path variants vs the previous kernel
for rep in 1 2; do
for v in spold default sp3nh sp2s3 sp2s2 sp2nh; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v $(PROBE_CONFIG=c2 timeout 600 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
done; done
