for rep in 1 2; do for v in default ma0; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "c3 $v $(PROBE_CONFIG=c3 PROBE_SIZES=1 timeout 600 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1)"
done; done
