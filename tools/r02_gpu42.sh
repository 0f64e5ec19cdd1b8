TOOLS="memcheck synccheck initcheck" bash tools/sanitize.sh
for t in memcheck synccheck initcheck; do echo "== $t"; grep "ERROR SUMMARY\|passed\|failed" gpurun_out/sanitize_$t.log; done
python tools/pcie_probe.py
