# after: straight-line single pass in quantize.cu (2 CTAs x 3 stages), permute+multiply code packing
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest4.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02_pytest4.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench6.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench6.log
