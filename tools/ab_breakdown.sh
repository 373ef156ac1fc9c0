# Same-box A/B (new build vs libbzg_v000.so) of cfg5 100k with the per-kernel breakdown.
cd $GRAFT_REPO_ROOT
L=paper_2411_13507_b200
cp $L/libbzg.so $L/libbzg_new.so
run() { python bench.py --config cfg5 --nodes 100000 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_breakdown_pass']
print('$1', round(d['ms_per_step'],3), 'sum', round(sum(k.values()),3), d['step_ms'], sorted(k.items(), key=lambda x:-x[1])[:8], d.get('host_phase_ms_last_step'))"; }
run new; cp $L/libbzg_v000.so $L/libbzg.so; run old; cp $L/libbzg_new.so $L/libbzg.so; run new
