for v in default ws_cap1 ws_c16s2p4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  timeout 600 python tools/with_variant.py $L -- bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-adapt > gpurun_out/r02_b16_$v.log 2>&1
  python tools/bl.py gpurun_out/r02_b16_$v.log
done
