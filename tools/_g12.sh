timeout 600 python tools/iter_cost.py cc22 > gpurun_out/g12_cc.txt 2>&1
WG_SPARSE_LOOP=0 timeout 600 python tools/iter_cost.py cc22 > gpurun_out/g12_cc_nosparse.txt 2>&1
timeout 600 python tools/iter_cost.py bfs16 > gpurun_out/g12_bfs16.txt 2>&1
WG_SPARSE_LOOP=0 timeout 600 python tools/iter_cost.py bfs16 > gpurun_out/g12_bfs16_nosparse.txt 2>&1
