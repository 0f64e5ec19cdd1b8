for v in default ws_c16s2p4 default ws_c16s2p4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  timeout 600 python tools/with_variant.py $L -- bench.py --config c3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-adapt --no-side > gpurun_out/r02_b17_$v.log 2>&1
  python tools/bl.py gpurun_out/r02_b17_$v.log
done
