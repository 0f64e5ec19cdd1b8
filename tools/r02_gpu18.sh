python __graft_entry__.py > gpurun_out/r02_smoke2.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 -p no:cacheprovider > gpurun_out/r02_pytest2.log 2>&1; echo pytest=$?; tail -14 gpurun_out/r02_pytest2.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench4.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench4.log
bash tools/make_profiles.sh r02
bash tools/sanitize.sh
for t in memcheck racecheck synccheck initcheck; do echo "== $t"; grep "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/sanitize_$t.log; done
