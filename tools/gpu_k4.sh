set -x
python -m pytest tests -x -q -m gpu 2>&1 | tail -5
for cfg in 0 4; do for w in cc22 sssp26 bfs26; do
WG_TMA_CFG=$cfg timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$w', d['ms_per_step'], d.get('config',{}).get('digest'), d.get('certificate'), d.get('phases'))"
done; done
