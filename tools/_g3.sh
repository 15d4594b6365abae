timeout 300 ./tools/mbsb > gpurun_out/g3_mbsb.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g3_parity.log
