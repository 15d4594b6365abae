timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/g19_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g19_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g19_bench.json 2> gpurun_out/g19_bench.err
WG_GRAPH=0 timeout 900 ncu -f --set full --import-source on -k regex:dense_dst --launch-skip 6 -c 3 -o /tmp/g19_cc python tools/prof_run.py cc22 2 > gpurun_out/g19_ncu.log 2>&1
ncu -i /tmp/g19_cc.ncu-rep --page details --csv > gpurun_out/g19_cc_details.csv 2>&1
ncu -i /tmp/g19_cc.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum > gpurun_out/g19_cc_raw.csv 2>&1
