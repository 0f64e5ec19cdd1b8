#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"allocate_kernel" -s 2 -c 1 \
  -o gpurun_out/r02_k2_4096 python tools/k2_once.py 4096 > gpurun_out/s52_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/s52_ncu.log
