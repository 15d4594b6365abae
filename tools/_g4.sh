timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_reference_suites.py > gpurun_out/g4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g4_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err
WG_DST_MAJOR=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g4_bench_old.json 2> gpurun_out/g4_bench_old.err
timeout 600 python bench.py --workload bfs26 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g4_bfs26.json 2> gpurun_out/g4_bfs26.err
