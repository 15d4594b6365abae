for i in 1 2 3; do for w in cc22; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], d['value'], d['parity']['ok'], d['clocks'], d['roofline']['kernel_sum_ms'])"
done; done
