V=paper_2104_14129_b200/csrc/build/var
for rep in 1 2; do for m in 1 2 3; do
timeout 300 python tools/with_variant.py $PWD/$V/libactnn_c8_s3_b2_p2_l-1_m$m.so -- bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('m$m', round(d['value'],1), round(d['ms_per_step'],3), {k:(round(v['ms_per_step'],3), round(v['frac'],3)) for k,v in d['roofline']['per_kernel'].items()})"
done; done
