#!/bin/bash
# Under gpurun: compute-sanitizer over small GPU parity tests (memcheck over the
# quantiser/dequantiser, contexts and NEXT-3 kernels; racecheck + synccheck over
# the kernels that share memory between warps).  Writes gpurun_out/sanitize_<tool>.log.
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_Q='c1_golden or adversarial_all_widths or ragged or unaligned or empty or mixed_widths_multi_tile'
SEL_A='grad_sqnorm_edges or ema or stale or ties_and_edges or resnet50_parity'
SEL_C='relu_pack_and_backward and 1023 or maxpool_forward_backward'
for tool in memcheck racecheck synccheck; do
  {
    echo "## $tool"
    timeout 1500 $CS --tool $tool --print-limit 20 python -m pytest -q -x tests/test_gpu_parity.py -k "$SEL_Q" 2>&1 | tail -4
    timeout 1500 $CS --tool $tool --print-limit 20 python -m pytest -q -x tests/test_gpu_adapt.py -k "$SEL_A" 2>&1 | tail -4
    timeout 1500 $CS --tool $tool --print-limit 20 python -m pytest -q -x tests/test_gpu_contexts.py -k "$SEL_C" 2>&1 | tail -4
  } > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool done"
done
