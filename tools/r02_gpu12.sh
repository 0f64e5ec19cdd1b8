for v in default dq_noswz default dq_noswz; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v c3 $(PROBE_CONFIG=c3 timeout 300 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1)"
done
