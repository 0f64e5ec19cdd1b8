#!/bin/bash
# K4 fixed cost per launch: end-of-CTA wait on the bulk stores' reads only (default)
# vs full completion (er0); TMA-store from 40 MB; 4-warp TMA-store CTAs (2 / 3 per SM).
for rep in 1 2; do for v in default er0 ts40 tsw4 tsw4o2; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "c3 $v $(PROBE_CONFIG=c3 PROBE_SIZES=1 timeout 600 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -2 | tr '\n' ' ')"
done; done
