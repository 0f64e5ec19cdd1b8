#!/bin/bash
# Stream-overlap evidence: kernel timelines (torch.profiler / CUPTI) of the pipelined step.
timeout 600 python tools/step_timeline.py --config c3 --trace gpurun_out/r02_timeline_c3.json.gz > gpurun_out/tl_c3.log 2>&1; echo c3=$?
timeout 600 python tools/step_timeline.py --config c3 --dist > gpurun_out/tl_c3_dist.log 2>&1; echo c3dist=$?
timeout 900 python tools/step_timeline.py --config c4 --trace gpurun_out/r02_timeline_c4.json.gz > gpurun_out/tl_c4.log 2>&1; echo c4=$?
for f in gpurun_out/tl_*.log; do echo "== $f"; tail -c 3000 $f; echo; done
