timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/g26_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g26_pytest.log
timeout 600 python bench.py --sharded --steps 5 --warmup 3 > gpurun_out/g26_sharded.json 2> gpurun_out/g26_sharded.err
