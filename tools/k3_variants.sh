#!/bin/bash
# Build libactnn variants of K3 (stage count / CTAs per SM / key mode) for a timing sweep.
cd "$(dirname "$0")/../paper_2104_14129_b200/csrc"
NV=/usr/local/cuda/bin/nvcc
A="-gencode arch=compute_100a,code=sm_100a"
mkdir -p build/var
for v in "3 2 0" "3 2 1" "2 3 0" "2 3 1" "4 1 0" "2 2 0" "5 1 0"; do
  set -- $v
  tag="s$1_b$2_k$3"
  $NV -O3 -std=c++17 $A -lineinfo -fmad=false -Xcompiler -fPIC -DACTNN_Q_S32=$1 -DACTNN_Q_MINB32=$2 -DACTNN_Q_KEYS=$3 -c quantize.cu -o build/var/q_$tag.o 2> build/var/q_$tag.txt &
done
wait
for f in build/var/q_*.o; do tag=$(basename $f .o | sed s/^q_//); $NV $A -shared -o build/var/libactnn_$tag.so build/abi.o $f build/dequantize.o build/stats.o build/allocate.o; echo "$tag $(grep -E 'Used' build/var/q_$tag.txt | sed -n '6p;8p' | grep -o 'Used [0-9]* reg' | tr '\n' ' ') $(grep -o '[0-9]* bytes spill stores' build/var/q_$tag.txt | sort -n | tail -1)"; done
