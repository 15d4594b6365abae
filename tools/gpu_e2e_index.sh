# e2e per index mode (placed vs chunked sort)
for w in ${WLS:-bfs26 sssp26}; do
  for m in placed sorted; do
    WG_E2E_INDEX=$m timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w $m', d['ms_per_step'], e['ms_per_step'], e['value'], e['h2d_bytes_per_step'], e.get('result_equal'), d['parity'].get('ok'))"
  done
done
