export WG_GRAPH=0
for w in cc22 sssp26; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$w.csv python tools/prof_run.py $w > /dev/null 2>&1
done
