for v in default q_s3m2 q_s4m2 q_s2m2 q_s3m3 default; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v c2 $(PROBE_CONFIG=c2 timeout 300 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
done
