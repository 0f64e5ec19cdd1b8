#!/bin/bash
# Variants of the warp-specialised K3 (consumers / stages / CTAs per SM) for tools/run_sweep.sh
cd "$(dirname "$0")/../paper_2104_14129_b200/csrc"
NV=/usr/local/cuda/bin/nvcc; A="-gencode arch=compute_100a,code=sm_100a"
rm -rf build/var; mkdir -p build/var
for v in "8 3 2" "8 2 3" "4 3 4" "4 4 3" "8 4 1" "12 2 2" "6 3 3"; do
  set -- $v; tag="c$1_s$2_b$3"
  $NV -O3 -std=c++17 $A -lineinfo -fmad=false -Xcompiler -fPIC -Xptxas -v -DACTNN_WS_CONS=$1 -DACTNN_WS_S=$2 -DACTNN_WS_MINB=$3 -c quantize_ws.cu -o build/var/w_$tag.o 2> build/var/w_$tag.txt &
done; wait
for f in build/var/w_*.o; do tag=$(basename $f .o | sed s/^w_//); $NV $A -shared -o build/var/libactnn_$tag.so build/abi.o build/quantize.o $f build/dequantize.o build/stats.o build/allocate.o; echo "$tag $(grep -E 'Used|spill' build/var/w_$tag.txt | paste - - | grep -o 'Used [0-9]* reg\|[0-9]* bytes spill stores' | tr '\n' ' ')"; done
