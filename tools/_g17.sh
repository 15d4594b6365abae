timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_reference_suites.py > gpurun_out/g17_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g17_pytest.log
for w in cc22 bfs16 bfs26 sssp26 sssp_grid pr25; do
timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g17_$w.json 2> gpurun_out/g17_$w.err
done
