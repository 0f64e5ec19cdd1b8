#!/bin/bash
# Under gpurun: the ncu evidence committed under profiles/ (see tools/profile_summary.py).
# 1) launch list of one full C3 step (serialised, cold caches: compare SHARES),
# 2) --set full on the four kernels of the largest tensor (bn1 input, 822 MB fp32).
TAG=${1:-r01}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"group_stats|allocate|quantize|uniform" -s 428 -c 428 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py --steps 1 > gpurun_out/${TAG}_ncu_list.log 2>&1
echo list=$?
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"^quantize_|^dequantize_fast|^group_stats|^allocate" -s 4 -c 4 \
  -o gpurun_out/${TAG}_full python tools/profile_step.py --steps 1 --layers 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo full=$?
