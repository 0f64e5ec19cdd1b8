set -x
tools/cuda_checks/f32x2_miscompile > gpurun_out/r02_f32x2_repro.log 2>&1; echo repro=$?
timeout 900 python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_f32x2/libactnn.so -- -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16meta.py tests/test_gpu_full_parity.py -x -q -p no:cacheprovider -k "not c4_whole and not c3_whole" > gpurun_out/r02_f32x2.log 2>&1; echo f32x2=$?
tail -3 gpurun_out/r02_f32x2.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k api_validates > gpurun_out/r02_api.log 2>&1; echo api=$?; tail -3 gpurun_out/r02_api.log
for v in default f32x2; do
  L=paper_2104_14129_b200/libactnn.so; [ $v = f32x2 ] && L=paper_2104_14129_b200/csrc/build/var_f32x2/libactnn.so
  for c in c3 c4; do
    timeout 600 python tools/with_variant.py $L -- bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-adapt > gpurun_out/r02_b_${v}_$c.log 2>&1
    python tools/bl.py gpurun_out/r02_b_${v}_$c.log
  done
done
bash tools/sanitize.sh
tail -8 gpurun_out/sanitize_*.log
