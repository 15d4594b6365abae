timeout 600 python tools/timeline.py cc22 > gpurun_out/g21_cc.txt 2>&1
