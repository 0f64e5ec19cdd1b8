# ncu --set full of the software-pipelined single-pass K3 (quantize_sp.cu) on C2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^quantize_sp" -s 1 -c 1 \
  -o gpurun_out/r02_c2_sp python tools/profile_step.py --config c2 --steps 1 > gpurun_out/r02_ncu_c2sp.log 2>&1; echo c2sp=$?
