set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g2_parity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g2_smoke.log
timeout 1500 python -m pytest tests/test_gpu_reference_suites.py -x -q -s > gpurun_out/g2_refsuites.log 2>&1; echo "rc=$?" >> gpurun_out/g2_refsuites.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
