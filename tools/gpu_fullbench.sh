# Round-end style measurement: default bench (+e2e, cpu_baseline), reference
# arm, every BASELINE config, and the ncu launch list of the default command
# (per-iteration launches: kernels inside conditional graphs cannot be profiled).
mkdir -p gpurun_out/full
python bench.py > gpurun_out/full/bench_cc22.json 2> gpurun_out/full/bench_cc22.err
python bench.py --impl reference > gpurun_out/full/reference_cc22.json 2> gpurun_out/full/reference_cc22.err
for w in bfs16 sssp_grid pr25 bfs26 sssp26; do
  timeout 900 python bench.py --workload $w > gpurun_out/full/bench_$w.json 2> gpurun_out/full/bench_$w.err
done
WG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/full/ncu_launches_cc22.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/full/ncu_bench.log 2>&1
ls -la gpurun_out/full
