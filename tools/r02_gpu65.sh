#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adapt.py tests/test_gpu_full_parity.py -q -x -k "allocate or mixed or virtual or stage or uncached or c2" > gpurun_out/s65_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/s65_pytest.log
timeout 300 python tools/k2_latency.py | cut -c80-400
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"group_stats|allocate|quantize|uniform|dequantize" -s 428 -c 428 --csv \
  --log-file gpurun_out/r02_launches.csv python tools/profile_step.py --steps 1 > gpurun_out/r02_ncu_list.log 2>&1
echo list=$?
