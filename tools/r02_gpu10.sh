timeout 1200 python -m pytest tests/test_gpu_full_parity.py -x -q -p no:cacheprovider > gpurun_out/r02_full_parity2.log 2>&1; echo fullparity=$?; tail -2 gpurun_out/r02_full_parity2.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench3.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench3.log
timeout 900 ncu --replay-mode app-range --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python tools/step_dram.py > gpurun_out/r02_step_dram.log 2>&1; echo dram=$?
tail -8 gpurun_out/r02_step_dram.log
timeout 900 ncu --replay-mode app-range --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python tools/step_dram.py --graph > gpurun_out/r02_step_dram_graph.log 2>&1; echo dramg=$?
tail -8 gpurun_out/r02_step_dram_graph.log
