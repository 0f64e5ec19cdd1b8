# round-2 evidence refresh, summarised on the box (the .ncu-rep files exceed gpurun's 64 MiB return limit)
bash tools/make_profiles.sh r02
python tools/profile_summary.py r02 > gpurun_out/r02_profile_summary.log 2>&1; echo summary=$?
bash tools/r02_prof1.sh
{ echo "# ncu --set full --clock-control none (tools/r02_prof1.sh), round 2 final kernels: C4 largest tensor K3 (bf16, warp-specialised), C3 largest tensor K4 (fp32, TMA-store path), C2 single-pass K3 (fp32, uniform 2-bit, straight-line full units).  Summaries by tools/ncu_brief.py."; python tools/ncu_brief.py gpurun_out/r02_c4_k3.ncu-rep gpurun_out/r02_c3_k4.ncu-rep gpurun_out/r02_c2_k3.ncu-rep; } > profiles/r02_ncu_full.txt
for k in c4_k3 c2_k3; do ncu -i gpurun_out/r02_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_${k}_sass.csv 2>/dev/null; done
mkdir -p gpurun_out/prof
cp profiles/r02_launches.csv profiles/r02_full.txt profiles/r02_c4_full.txt profiles/r02_adapt_full.txt profiles/traffic.json profiles/r02_ncu_full.txt gpurun_out/prof/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/prof; du -sh gpurun_out
