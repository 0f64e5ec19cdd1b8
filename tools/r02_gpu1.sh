set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
nproc; free -g | head -2
python __graft_entry__.py > gpurun_out/r02_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=20 -p no:cacheprovider > gpurun_out/r02_pytest1.log 2>&1; echo pytest=$?
tail -30 gpurun_out/r02_pytest1.log
timeout 600 python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_f32x2/libactnn.so -- -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16meta.py -x -q -k "adversarial or mixed_widths or ragged or philox or full_size or uncached" -p no:cacheprovider > gpurun_out/r02_f32x2.log 2>&1; echo f32x2=$?
tail -3 gpurun_out/r02_f32x2.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02_bench1.log 2>&1; echo bench=$?
tail -c 1500 gpurun_out/r02_bench1.log
