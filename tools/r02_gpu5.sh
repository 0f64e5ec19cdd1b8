timeout 600 python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_ts/libactnn.so -- -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16meta.py tests/test_gpu_full_parity.py -x -q -p no:cacheprovider -k "not c4_whole and not c3_whole" > gpurun_out/r02_ts_parity.log 2>&1; echo ts_parity=$?; tail -2 gpurun_out/r02_ts_parity.log
for v in default ts ts_o3 ts_s6 ts_o3s6 ts_o4s3; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  for c in c3 c4; do
    echo "$v $c $(PROBE_CONFIG=$c timeout 300 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1)"
  done
done
