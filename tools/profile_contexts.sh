#!/bin/bash
# Under gpurun: ncu --set full of the NEXT-4 context kernels -> gpurun_out/<tag>_contexts.ncu-rep
TAG=${1:-r01}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"maxpool|relu" -c 10 \
    -o gpurun_out/${TAG}_contexts python tools/contexts_once.py > gpurun_out/${TAG}_contexts_ncu.log 2>&1
echo ncu=$?
