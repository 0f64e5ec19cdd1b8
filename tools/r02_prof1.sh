# ncu --set full on: C4 largest tensor's K3 (bf16 warp-specialised), C3 largest
# tensor's K4 (fp32, TMA-store), C2's single-pass K3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^quantize_ws" -s 1 -c 1 \
  -o gpurun_out/r02_c4_k3 python tools/profile_step.py --config c4 --steps 1 --layers 1 > gpurun_out/r02_ncu_c4k3.log 2>&1; echo c4k3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^dequantize_fast" -s 1 -c 1 \
  -o gpurun_out/r02_c3_k4 python tools/profile_step.py --config c3 --steps 1 --layers 1 > gpurun_out/r02_ncu_c3k4.log 2>&1; echo c3k4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^quantize_sp8" -s 1 -c 1 \
  -o gpurun_out/r02_c2_k3 python tools/profile_step.py --config c2 --steps 1 > gpurun_out/r02_ncu_c2k3.log 2>&1; echo c2k3=$?
ls -la gpurun_out/*.ncu-rep
