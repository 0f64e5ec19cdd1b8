TOOLS=synccheck bash tools/sanitize.sh
grep "ERROR SUMMARY\|passed\|failed\|Warning" gpurun_out/sanitize_synccheck.log
bash tools/r02_gpu36.sh
./tools/cuda_checks/k3_mix | grep -E "warps/SM=32" | grep -E "split|lop_2ffma|wide_2ffma|m_wide |m_lop "
