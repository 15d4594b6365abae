timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/g24_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g24_pytest.log
