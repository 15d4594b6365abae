python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cc22.json 2>gpurun_out/bench_cc22.err
tail -c 300 gpurun_out/bench_cc22.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cc22.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
WG_GRAPH=0 ncu --set full --import-source on --clock-control none -k regex:pull_dense_tma --launch-skip 1 -c 1 -o /tmp/dense_cc22 python tools/prof_run.py cc22 > /dev/null 2>&1
ncu -i /tmp/dense_cc22.ncu-rep --page raw --csv > gpurun_out/dense_cc22_raw.csv
ncu -i /tmp/dense_cc22.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/dense_cc22_source.csv 2>/dev/null || ncu -i /tmp/dense_cc22.ncu-rep --page source --csv > gpurun_out/dense_cc22_source.csv
ncu -i /tmp/dense_cc22.ncu-rep --page details > gpurun_out/dense_cc22_details.txt
ls -la gpurun_out
