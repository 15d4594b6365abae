for w in sssp26 bfs26 cc22; do for cfg in 1 2 3 4; do
WG_TMA_CFG=$cfg timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$w', d['ms_per_step'], d['parity'], [x['pull_ms'] for x in d['roofline']['per_iteration'] if x['mode']=='FullScan'])"
done; done
