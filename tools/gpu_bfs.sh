python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for w in bfs26 bfs16 cc22 sssp26; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], d['value'], d['parity'], [(x['mode'][0], x['pull_ms'], x['prep_ms'], x['end_ms']) for x in d['roofline']['per_iteration']])"
done
