# fp32 single pass on 8-group units (12 warps), PDL: full suite, bench
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest6.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02_pytest6.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench9.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench9.log
