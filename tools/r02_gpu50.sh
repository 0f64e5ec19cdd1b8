#!/bin/bash
# Kernel timelines of the pipelined step (C3, C3 multi-rank path, C4) + a default bench line
# (now with the K2 latency fields).
timeout 600 python tools/step_timeline.py --config c3 --trace gpurun_out/r02_timeline_c3.json.gz > gpurun_out/tl_c3.log 2>&1; echo c3=$?
timeout 600 python tools/step_timeline.py --config c3 --dist > gpurun_out/tl_c3_dist.log 2>&1; echo c3dist=$?
timeout 900 python tools/step_timeline.py --config c4 --trace gpurun_out/r02_timeline_c4.json.gz > gpurun_out/tl_c4.log 2>&1; echo c4=$?
timeout 900 python bench.py > gpurun_out/s50_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/s50_bench_c3.log | cut -c1-300
