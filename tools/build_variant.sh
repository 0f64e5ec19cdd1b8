#!/bin/bash
# Build an alternative libactnn.so with extra -D flags (tuning / diagnostics only):
#   tools/build_variant.sh TAG "-DACTNN_WIDE_F32X2=1 ..."
# -> paper_2104_14129_b200/csrc/build/var_TAG/libactnn.so.  Load it with
#   python tools/with_variant.py paper_2104_14129_b200/csrc/build/var_TAG/libactnn.so -- <script|-m mod> args
set -e
TAG=$1; shift; FLAGS="$*"
cd "$(dirname "$0")/../paper_2104_14129_b200/csrc"
NV=/usr/local/cuda/bin/nvcc
A="-gencode arch=compute_100a,code=sm_100a"
D=build/var_$TAG
mkdir -p $D
for f in abi quantize quantize_ws quantize_sp8 dequantize stats allocate contexts adapt; do
  $NV -O3 -std=c++17 $A -lineinfo -fmad=false -Xcompiler -fPIC,-O2 -Xptxas -v $FLAGS -c $f.cu -o $D/$f.o 2> $D/$f.ptxas.txt &
done
wait
$NV $A -shared -o $D/libactnn.so $D/*.o && find $D -name "*.o" -delete
echo "$D/libactnn.so ($FLAGS)"
