for v in default ts8o4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  for c in c3 c4; do
    PROBE_DUMP=1 PROBE_CONFIG=$c timeout 300 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1 > gpurun_out/k4_${v}_$c.json
  done
done
