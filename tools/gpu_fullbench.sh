# Round-end style measurement: default bench (+e2e, cpu_baseline), reference
# arm, every BASELINE config, the ncu launch list of the default command
# (per-iteration launches: kernels inside conditional graphs cannot be
# profiled) and a full capture of the dominant kernel.
mkdir -p gpurun_out/full
python bench.py > gpurun_out/full/bench_cc22.json 2> gpurun_out/full/bench_cc22.err
python bench.py --impl reference > gpurun_out/full/reference_cc22.json 2> gpurun_out/full/reference_cc22.err
for w in bfs16 sssp_grid pr25 bfs26 sssp26; do
  timeout 900 python bench.py --workload $w > gpurun_out/full/bench_$w.json 2> gpurun_out/full/bench_$w.err
done
[ "${WITH_NCU:-1}" = 0 ] && { ls -la gpurun_out/full; exit 0; }
WG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/full/ncu_launches_cc22.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/full/ncu_bench.log 2>&1
WG_GRAPH=0 ncu --set full --import-source on --clock-control none -k regex:pull_dense_tma --launch-skip 1 -c 1 -o /tmp/dense_cc22 python tools/prof_run.py cc22 > /dev/null 2>&1
ncu -i /tmp/dense_cc22.ncu-rep --page raw --csv > gpurun_out/full/dense_cc22_raw.csv
ncu -i /tmp/dense_cc22.ncu-rep --page details > gpurun_out/full/dense_cc22_details.txt
ls -la gpurun_out/full
