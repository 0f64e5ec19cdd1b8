# K4: TMA-store warps/staging variants per output size (sequence timing)
for c in c3 c4; do for v in ts0 ts1 ts16o2 ts12o3; do
  L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$c $v $(PROBE_CONFIG=$c PROBE_SIZES=1 timeout 600 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1)"
done; done
