#!/bin/bash
# Under gpurun: the ncu evidence committed under profiles/ (see tools/profile_summary.py).
# 1) launch list of one full C3 step (serialised, cold caches: compare SHARES),
# 2) --set full on the kernels of the largest C3 tensor (bn1 input, 822 MB fp32),
# 3) --set full on the kernels of the largest C4 tensor (1.64 GB bf16),
# 4) --set full on the NEXT-3 kernels (K6 grad_sqnorm, K5 stage-2 allocation).
TAG=${1:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"group_stats|allocate|quantize|uniform|dequantize" -s 428 -c 428 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py --steps 1 > gpurun_out/${TAG}_ncu_list.log 2>&1
echo list=$?
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"^quantize_|^dequantize_fast|^group_stats|^allocate" -s 4 -c 4 \
  -o gpurun_out/${TAG}_full python tools/profile_step.py --steps 1 --layers 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo full=$?
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"^quantize_|^dequantize_fast|^group_stats|^allocate" -s 4 -c 4 \
  -o gpurun_out/${TAG}_c4_full python tools/profile_step.py --config c4 --steps 1 --layers 1 > gpurun_out/${TAG}_ncu_c4.log 2>&1
echo c4=$?
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"grad_sqnorm|allocate_layers" \
  -o gpurun_out/${TAG}_adapt_full python tools/profile_adapt.py > gpurun_out/${TAG}_ncu_adapt.log 2>&1
echo adapt=$?
