timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench7.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench7.log
timeout 300 python -m pytest tests/test_bench_contract.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
