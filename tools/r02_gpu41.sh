TOOLS=racecheck bash tools/sanitize.sh
cat gpurun_out/sanitize_racecheck.log | grep -v "Host Frame" | grep -E "passed|failed|SUMMARY|Thread|###|mode" | head -60
