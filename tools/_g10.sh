for w in cc22 bfs26; do
  if [ $w = cc22 ]; then sk=7; else sk=8; fi
  WG_GRAPH=0 timeout 900 ncu -f --set full --import-source on -k regex:dense_dst --launch-skip $sk -c 1 -o /tmp/g10_$w python tools/prof_run.py $w 2 > gpurun_out/g10_ncu_$w.log 2>&1
  ncu -i /tmp/g10_$w.ncu-rep --page details --csv > gpurun_out/g10_${w}_details.csv 2>&1
  ncu -i /tmp/g10_$w.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/g10_${w}_source.csv 2>&1
done
