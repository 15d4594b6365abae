timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_reference_suites.py > gpurun_out/g20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g20_pytest.log
timeout 600 python tools/iter_cost.py cc22 > gpurun_out/g20_cc.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g20_bench.json 2> gpurun_out/g20_bench.err
timeout 600 python bench.py --workload bfs16 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g20_bfs16.json 2> gpurun_out/g20_bfs16.err
