python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for w in ${WLS:-sssp_grid cc22 sssp26 bfs26}; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['per_iteration']; print('$w', d['ms_per_step'], d['value'], d['parity'].get('digest'), d['parity'].get('ok'), d['parity'].get('certificate',{}).get('ok'), [(x['mode'][0], x['pull_ms'], x['prep_ms'], x['end_ms']) for x in r][:12])"
done
