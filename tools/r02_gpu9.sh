for v in default ws_csleep ws_c16p4sleep ws_m3ph1 ws_noswp ws_c16s3p4 ws_c16s2p4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  for c in c4 c3; do
    echo "$v $c $(PROBE_CONFIG=$c timeout 300 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
  done
done
