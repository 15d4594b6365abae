timeout 600 python tools/prof_persistent.py sssp_grid 2000 1000 > gpurun_out/g18_grid.txt 2>&1
WG_PERSIST_BLOCKS=1 timeout 600 python tools/prof_persistent.py sssp_grid 2000 1000 > gpurun_out/g18_grid_b1.txt 2>&1
WG_PERSIST_BLOCKS=2 timeout 600 python tools/prof_persistent.py sssp_grid 2000 1000 > gpurun_out/g18_grid_b2.txt 2>&1
