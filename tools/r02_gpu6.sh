for v in default ts8o2 ts8o3 ts12o3 ts16o2s3 ts4o3m2 ts8o4 ts6o4; do
  L=paper_2104_14129_b200/libactnn.so; [ $v != default ] && L=paper_2104_14129_b200/csrc/build/var_$v/libactnn.so
  for c in c3 c4; do
    echo "$v $c $(PROBE_CONFIG=$c timeout 300 python tools/with_variant.py $L -- tools/k4_probe.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v,3) if isinstance(v,float) else v for k,v in d.items()})')"
  done
done
