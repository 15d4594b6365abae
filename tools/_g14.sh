timeout 600 python tools/timeline.py cc22 > gpurun_out/g14_cc.txt 2>&1
timeout 600 python tools/timeline.py bfs16 > gpurun_out/g14_bfs16.txt 2>&1
