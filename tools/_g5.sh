timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g5_pytest.log
WG_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/g5_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g5_ncu.log 2>&1
