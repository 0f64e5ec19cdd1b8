set -x
TOOLS="racecheck initcheck" bash tools/sanitize.sh
cat gpurun_out/sanitize_racecheck.log | head -60
cat gpurun_out/sanitize_initcheck.log | head -30
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_bench_contract.py -q -x -p no:cacheprovider > gpurun_out/r02_dist.log 2>&1; echo dist=$?; tail -5 gpurun_out/r02_dist.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench2.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/r02_bench2.log
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_bench_c5k1.log 2>&1; echo c5=$?
tail -c 1500 gpurun_out/r02_bench_c5k1.log
