# e2e lines of the given workloads for each upload format + GPU parity tests
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for w in ${WLS:-cc22 bfs16 sssp26}; do
  for f in ${FMTS:-coded bits raw}; do
    WG_E2E_FORMAT=$f timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/e2e_err_$w_$f.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w $f', d['ms_per_step'], e['ms_per_step'], e['value'], e['h2d_bytes_per_step'], e.get('lane_bits_per_lane'), e.get('result_equal'), e.get('host_format_build_s'), d['parity'].get('ok'))"
  done
done
