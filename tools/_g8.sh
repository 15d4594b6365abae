for w in cc22 bfs26; do
WG_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum -k regex:dense_dst -c 40 --csv python tools/prof_run.py $w 2 > gpurun_out/g8_seq_$w.csv 2>&1
done
