export WG_GRAPH=0
ncu --set full --import-source on --clock-control none -k regex:pull_kernel --launch-skip 1 -c 1 -o /tmp/bfs26 python tools/prof_run.py bfs26 > gpurun_out/bfsprof_run.log 2>&1
ncu -i /tmp/bfs26.ncu-rep --page raw --csv > gpurun_out/bfs26_raw.csv
ncu -i /tmp/bfs26.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/bfs26_source.csv
ncu -i /tmp/bfs26.ncu-rep --page details > gpurun_out/bfs26_details.txt
