timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_reference_suites.py > gpurun_out/g22_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g22_pytest.log
timeout 600 python tools/timeline.py cc22 > gpurun_out/g22_cc.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g22_bench.json 2> gpurun_out/g22_bench.err
for w in bfs16 bfs26 sssp26; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g22_$w.json 2> gpurun_out/g22_$w.err; done
