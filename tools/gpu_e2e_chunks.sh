# e2e (coded upload) per chunk count
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for w in ${WLS:-cc22 sssp26}; do
  for c in ${CHUNKS:-4 6 8}; do
    WG_E2E_CHUNKS=$c timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w chunks=$c', d['ms_per_step'], e['ms_per_step'], e['value'], e['h2d_bytes_per_step'], e.get('result_equal'), d['parity'].get('ok'))"
  done
done
