timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest_pack2.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02_pytest_pack2.log
./tools/cuda_checks/k3_mix | grep "b1 "
