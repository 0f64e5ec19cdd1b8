# racecheck hazard sites: TMA-store K4 test alone, then the uncached-variants test (details, source lines)
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_full_parity.py -k "tma_store_dequantize_large_fp32 and 2048" > gpurun_out/race_k4ts.log 2>&1
tail -3 gpurun_out/race_k4ts.log
grep -A1 -E "(Write|Read) Thread" gpurun_out/race_k4ts.log | grep -oE "[a-z_0-9]+\.cu:[0-9]+" | sed -E 's/Thread \([0-9,]+\) at //; s/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -20
timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_full_parity.py -k "uncached_variants_n4100 and 1280" > gpurun_out/race_unc.log 2>&1
tail -3 gpurun_out/race_unc.log
grep -A1 -E "(Write|Read) Thread" gpurun_out/race_unc.log | grep -oE "[a-z_0-9]+\.cu:[0-9]+" | sed -E 's/Thread \([0-9,]+\) at //; s/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -20
