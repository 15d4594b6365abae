export WG_GRAPH=0
for cfg in 0 4; do
WG_TMA_CFG=$cfg ncu --metrics gpu__time_duration.sum,smsp__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pull_dense --csv --log-file gpurun_out/k4_launch_sssp26_$cfg.csv python tools/prof_run.py sssp26 > /dev/null 2>&1
WG_TMA_CFG=$cfg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pull_dense --csv --log-file gpurun_out/k4_launch_cc22_$cfg.csv python tools/prof_run.py cc22 > /dev/null 2>&1
done
WG_TMA_CFG=0 ncu --set full --import-source on --clock-control none -k regex:pull_dense_k4 --launch-skip 3 -c 1 -o gpurun_out/k4_sssp26 python tools/prof_run.py sssp26 > /dev/null 2>&1
WG_TMA_CFG=4 ncu --set full --import-source on --clock-control none -k regex:pull_dense_tma --launch-skip 3 -c 1 -o gpurun_out/tma_sssp26 python tools/prof_run.py sssp26 > /dev/null 2>&1
ls -la gpurun_out
