timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16meta.py tests/test_gpu_full_parity.py tests/test_gpu_contexts.py tests/test_gpu_adapt.py -x -q -p no:cacheprovider -k "not c4_whole and not c3_whole" > gpurun_out/r02_uws_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/r02_uws_parity.log
for v in default uws0 default uws0; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v c2 $(PROBE_CONFIG=c2 timeout 300 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
done
