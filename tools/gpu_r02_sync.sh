timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for cfg in cfg1 cfg2 cfg3; do timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_breakdown_pass']
print('$cfg', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'launches', d['gpu_launches_per_step'], 'ksum', round(sum(k.values()),4), d.get('host_phase_ms_last_step'))"; done
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-600
