# GPU tests + per-iteration pull times of the given workloads
python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for w in ${WLS:-cc22 sssp26}; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], d['value'], d['parity'].get('ok'), [(r['mode'][0], r['pull_ms']) for r in d['roofline']['per_iteration']][:8])"
done
