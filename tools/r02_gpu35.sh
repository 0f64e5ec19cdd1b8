# sanitizers over the round-2 final kernels (PDL launches, permute+multiply packing, straight-line single pass)
bash tools/sanitize.sh
for t in memcheck racecheck synccheck initcheck; do echo "== $t"; grep "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/sanitize_$t.log; done
