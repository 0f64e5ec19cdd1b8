#!/bin/bash
# Variants of the warp-specialised K3 for tools/run_sweep.sh.
# WS_VARIANTS="cons stages minblocks philox_batch lazy meta_depth|..." (| separated)
cd "$(dirname "$0")/../paper_2104_14129_b200/csrc"
NV=/usr/local/cuda/bin/nvcc; A="-gencode arch=compute_100a,code=sm_100a"
rm -rf build/var; mkdir -p build/var
IFS='|' read -ra VARS <<< "${WS_VARIANTS:-8 3 2 2 -1 1}"
for v in "${VARS[@]}"; do
  set -- $v; tag="c$1_s$2_b$3_p$4_l$5_m${6:-1}"
  $NV -O3 -std=c++17 $A -lineinfo -fmad=false -Xcompiler -fPIC -Xptxas -v -DACTNN_WS_CONS=$1 \
      -DACTNN_WS_S=$2 -DACTNN_WS_MINB=$3 -DACTNN_WS_PH=$4 -DACTNN_WS_LAZY=$5 -DACTNN_WS_MD=${6:-1} \
      -c quantize_ws.cu -o build/var/w_$tag.o 2> build/var/w_$tag.txt &
done; wait
for f in build/var/w_*.o; do
  tag=$(basename $f .o | sed s/^w_//)
  $NV $A -shared -o build/var/libactnn_$tag.so $(ls build/*.o | grep -v quantize_ws) $f
  echo "$tag $(grep -E 'Used|spill' build/var/w_$tag.txt | paste - - | grep -o 'Used [0-9]* reg\|[0-9]* bytes spill stores' | tr '\n' ' ')"
done
