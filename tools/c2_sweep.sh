#!/bin/bash
# Under gpurun: C2 bench (uniform single pass) for every variant library in build/$VARDIR.
for f in paper_2104_14129_b200/csrc/build/${VARDIR:-v17}/libactnn_*.so; do
  echo "$(basename $f)"; timeout 300 python tools/with_variant.py $PWD/$f -- bench.py --config c2 --steps 20 --no-cpu --no-e2e > /tmp/c2v.log 2>&1; python tools/bl.py /tmp/c2v.log
done
timeout 300 python bench.py --config c2 --steps 20 --no-cpu --no-e2e > /tmp/c2v.log 2>&1; echo default; python tools/bl.py /tmp/c2v.log
