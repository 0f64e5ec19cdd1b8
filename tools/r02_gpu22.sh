# single-pass software-pipelined K3 (quantize_sp.cu): parity, then timing variants
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c4_whole_step" > gpurun_out/r02_pytest_sp.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02_pytest_sp.log
for rep in 1 2; do
for v in nosp default spB spC spD; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$v $(PROBE_CONFIG=c2 timeout 600 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
done; done
