timeout 600 python tools/iter_cost.py bfs26 3 > gpurun_out/g16_bfs26.txt 2>&1
WG_LOOP_DENSE=0 timeout 600 python tools/iter_cost.py bfs26 3 > gpurun_out/g16_bfs26_nold.txt 2>&1
WG_LOOP_DENSE=0 timeout 600 python tools/iter_cost.py cc22 > gpurun_out/g16_cc_nold.txt 2>&1
