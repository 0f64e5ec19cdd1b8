#!/bin/bash
# Time every variant library in build/var plus the default build (tools/kernel_sweep.py).
for f in paper_2104_14129_b200/csrc/build/${VARDIR:-var}/libactnn_*.so; do
  timeout 300 python tools/with_variant.py $PWD/$f -- tools/kernel_sweep.py 2>&1 | tail -1
done
timeout 300 python tools/kernel_sweep.py 2>&1 | tail -1
