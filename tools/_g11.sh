timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x > gpurun_out/g11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g11_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g11_bench.json 2> gpurun_out/g11_bench.err
timeout 600 python bench.py --workload bfs26 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g11_bfs26.json 2> gpurun_out/g11_bfs26.err
