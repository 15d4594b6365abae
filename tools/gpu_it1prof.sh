export WG_GRAPH=0
ncu --set full --import-source on --clock-control none -k regex:pull_dense_tma --launch-skip 0 -c 1 -o /tmp/it1 python tools/prof_run.py cc22 > /dev/null 2>&1
ncu -i /tmp/it1.ncu-rep --page raw --csv > gpurun_out/it1_raw.csv
ncu -i /tmp/it1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/it1_source.csv
