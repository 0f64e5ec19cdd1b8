timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16meta.py tests/test_gpu_full_parity.py -x -q -p no:cacheprovider -k "not c4_whole and not c3_whole" > gpurun_out/r02_fhadd_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/r02_fhadd_parity.log
for v in pre_fhadd default ws_c16s2 ws_c16s2p4 ws_ph4 ws_ph1 ws_m3s2; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  for c in c4 c3; do
    echo "$v $c $(PROBE_CONFIG=$c timeout 300 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
  done
done
