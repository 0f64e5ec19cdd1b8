#!/bin/bash
timeout 900 python bench.py > gpurun_out/s76_bench_c3.log 2>&1; echo c3=$?
python tools/bl.py gpurun_out/s76_bench_c3.log
tail -1 gpurun_out/s76_bench_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['adapt']['grad_sqnorm']))"
timeout 1500 python bench.py --config c5 --steps 5 --no-cpu --no-e2e > gpurun_out/s76_bench_c5.log 2>&1; echo c5=$?
python tools/bl.py gpurun_out/s76_bench_c5.log
timeout 600 python -m pytest tests/test_bench_contract.py -q 2>&1 | tail -1
