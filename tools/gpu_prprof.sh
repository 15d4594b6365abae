for v in 0 1; do
WG_PR_DIRECT=$v ncu --set full --clock-control none -k regex:pr_pull --launch-skip 3 -c 1 -o /tmp/pr$v python tools/prof_run.py pr25 > /dev/null 2>&1
ncu -i /tmp/pr$v.ncu-rep --page raw --csv > gpurun_out/pr$v.csv
done
