timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_reference_suites.py > gpurun_out/g9_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g9_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err
timeout 600 python bench.py --workload bfs26 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g9_bfs26.json 2> gpurun_out/g9_bfs26.err
timeout 600 python bench.py --workload bfs16 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g9_bfs16.json 2> gpurun_out/g9_bfs16.err
