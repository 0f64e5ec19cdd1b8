# K4 metadata by cp.async + mbarrier arrive (kMA) instead of two bulk copies: parity subset, per-size timing
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c1 or adversarial or ragged or bf16meta or empty or unaligned or uncached or mixed_widths or tma_store or c2 or dequant or whole_step" > gpurun_out/r02_pytest_ma.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02_pytest_ma.log
for c in c3 c4; do for v in ma0 default; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  echo "$c $v $(PROBE_CONFIG=$c PROBE_SIZES=1 timeout 600 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1)"
done; done
