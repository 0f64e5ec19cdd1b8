# byte-permute + multiply code packing (ACTNN_PACK_MUL): parity subset, then K3 timing vs the shift/mask packing
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c4_whole_step" > gpurun_out/r02_pytest_pack.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02_pytest_pack.log
for rep in 1 2; do
for c in c4 c3 c2; do
for v in pack0 default; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$c $v $(PROBE_CONFIG=$c timeout 600 python tools/with_variant.py $L -- tools/k3_probe.py 2>&1 | tail -1)"
done; done; done
