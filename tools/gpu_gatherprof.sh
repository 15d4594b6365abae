export WG_GRAPH=0
for go in 0 1; do
WG_GATHER_ORDER=$go ncu --set full --clock-control none -k regex:pull_dense_tma --launch-skip 2 -c 1 -o /tmp/go${go}_sssp26 python tools/prof_run.py sssp26 > /dev/null 2>&1
WG_GATHER_ORDER=$go ncu --set full --clock-control none -k regex:pull_dense_tma --launch-skip 1 -c 1 -o /tmp/go${go}_cc22 python tools/prof_run.py cc22 > /dev/null 2>&1
ncu -i /tmp/go${go}_sssp26.ncu-rep --page raw --csv > gpurun_out/go${go}_sssp26.csv
ncu -i /tmp/go${go}_cc22.ncu-rep --page raw --csv > gpurun_out/go${go}_cc22.csv
done
ls -la gpurun_out
