ACTNN_LAYER_DUMP=gpurun_out/r02_layers_c3.json timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-adapt --no-side > gpurun_out/r02_b13.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_b13.log
