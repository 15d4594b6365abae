python tools/prof_persistent.py sssp_grid 2000 2000 > gpurun_out/grid_phases.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:sparse_loop --launch-skip 1 -c 1 -o /tmp/grid python tools/prof_persistent.py sssp_grid 300 2000 > gpurun_out/grid_ncu.log 2>&1
ncu -i /tmp/grid.ncu-rep --page raw --csv > gpurun_out/grid_raw.csv
ncu -i /tmp/grid.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/grid_source.csv
ncu -i /tmp/grid.ncu-rep --page details > gpurun_out/grid_details.txt
