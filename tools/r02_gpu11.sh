timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16meta.py tests/test_gpu_full_parity.py -x -q -p no:cacheprovider -k "not c4_whole and not c3_whole" > gpurun_out/r02_fastbf16_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/r02_fastbf16_parity.log
for v in default dq_u8ts dq_u8 dq_u8ts_o2; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v c4 $(PROBE_CONFIG=c4 timeout 300 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1)"
done
echo "dq_u8ts_o2 c3 $(PROBE_CONFIG=c3 timeout 300 python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_dq_u8ts_o2/libactnn.so -- tools/k4_probe.py 2>&1 | tail -1)"
echo "dq_u8 c3 $(PROBE_CONFIG=c3 timeout 300 python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_dq_u8/libactnn.so -- tools/k4_probe.py 2>&1 | tail -1)"
timeout 900 ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python tools/step_dram.py > gpurun_out/r02_step_dram.log 2>&1; echo dram=$?
tail -8 gpurun_out/r02_step_dram.log
