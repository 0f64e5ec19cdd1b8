# session 2 re-entry: confirm HEAD (16+4 warp-specialised K3) on a fresh box
python __graft_entry__.py > gpurun_out/r02_smoke3.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 -p no:cacheprovider > gpurun_out/r02_pytest3.log 2>&1; echo pytest=$?; tail -20 gpurun_out/r02_pytest3.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench5.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench5.log
