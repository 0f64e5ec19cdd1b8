# programmatic dependent launch on the hot-path kernels: full suite, bench, K4 per-size sequence
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest5.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02_pytest5.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench8.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench8.log
grep -o '"graph_error[^,]*' gpurun_out/r02_bench8.log | head -2
PROBE_CONFIG=c3 PROBE_SIZES=1 timeout 600 python tools/k4_probe.py 2>&1 | tail -1
