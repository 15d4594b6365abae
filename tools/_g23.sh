timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "pagerank or sharded" > gpurun_out/g23_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g23_pytest.log
timeout 900 python bench.py --workload pr25 --steps 3 --warmup 3 --no-e2e > gpurun_out/g23_pr25.json 2> gpurun_out/g23_pr25.err
