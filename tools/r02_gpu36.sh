# fp32 single pass on 8-group units (quantize_sp8.cu): parity subset, then C2 K3 timing variants
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c2 or c1 or adversarial or ragged or bf16meta or philox or empty or unaligned or uncached or mixed_widths" > gpurun_out/r02_pytest_sp8.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02_pytest_sp8.log
for rep in 1 2; do
for v in nosp8 default sp8w8 sp8w12 sp8s3; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "c2 $v $(PROBE_CONFIG=c2 timeout 600 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
done; done
