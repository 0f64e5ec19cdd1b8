# K3 bf16: looped SWP variants (ACTNN_WS_LOOP) vs default, C4 serial K3 probe
for rep in 1 2; do
for v in default loop loop1 loop4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v $(PROBE_CONFIG=c4 timeout 600 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
done; done
