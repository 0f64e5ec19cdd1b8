# round-2 evidence, final kernels: GPU suite, bench line (C3 + side legs), ncu launch list + --set full (summarised on the box)
python __graft_entry__.py > gpurun_out/r02_smoke_final.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_final.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r02_pytest_final.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_final.log 2>&1; echo bench=$?
python tools/bl.py gpurun_out/r02_bench_final.log
bash tools/make_profiles.sh r02
python tools/profile_summary.py r02 > gpurun_out/r02_profile_summary.log 2>&1; echo summary=$?
bash tools/r02_prof1.sh
{ echo "# ncu --set full --clock-control none (tools/r02_prof1.sh), round 2 final kernels: C4 largest tensor K3 (bf16, warp-specialised), C3 largest tensor K4 (fp32, TMA-store path), C2 single-pass K3 (fp32, 8-group units, quantize_sp8.cu).  Summaries by tools/ncu_brief.py."; python tools/ncu_brief.py gpurun_out/r02_c4_k3.ncu-rep gpurun_out/r02_c3_k4.ncu-rep gpurun_out/r02_c2_k3.ncu-rep; } > profiles/r02_ncu_full.txt
mkdir -p gpurun_out/prof
cp profiles/r02_launches.csv profiles/r02_full.txt profiles/r02_c4_full.txt profiles/r02_adapt_full.txt profiles/traffic.json profiles/r02_ncu_full.txt gpurun_out/prof/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
