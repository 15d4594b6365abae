
for w in cc22 bfs26; do
  if [ $w = cc22 ]; then sk=6; c=3; else sk=7; c=2; fi
  WG_GRAPH=0 timeout 900 ncu -f --set full --import-source on -k regex:dense_dst --launch-skip $sk -c $c -o /tmp/g7_$w python tools/prof_run.py $w 2 > gpurun_out/g7_ncu_$w.log 2>&1
  ncu -i /tmp/g7_$w.ncu-rep --page details --csv > gpurun_out/g7_${w}_details.csv 2>&1
  ncu -i /tmp/g7_$w.ncu-rep --page raw --csv > gpurun_out/g7_${w}_raw.csv 2>&1
  ncu -i /tmp/g7_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/g7_${w}_source.csv 2>&1
done
ls -la gpurun_out
