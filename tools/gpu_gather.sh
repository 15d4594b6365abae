python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for w in cc22 sssp26 sssp_grid pr25; do for go in 0 1; do
WG_GATHER_ORDER=$go timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('go=$go', '$w', d['ms_per_step'], d['parity'].get('digest'), d['parity'].get('ok'), d['parity'].get('certificate',{}).get('ok'), [x['pull_ms'] for x in d['roofline']['per_iteration'] if x['mode']=='FullScan'], [x['end_ms'] for x in d['roofline']['per_iteration'] if x['mode']=='FullScan'])"
done; done
