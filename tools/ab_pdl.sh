# Same-box A/B of programmatic dependent launch (BZG_PDL=1 default vs BZG_PDL=0), alternating.
#   gpurun -- 'CFGS="cfg1-demo cfg1 cfg2" bash tools/ab_pdl.sh'
cd ${GRAFT_REPO_ROOT:-.}
run() { BZG_PDL=$2 python bench.py --config $1 --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('eager') or {}; print('$1 pdl=$2', round(d['ms_per_step'],4), 'e2e', round((d.get('e2e') or {}).get('ms_per_step', (d.get('e2e') or {}).get('value', 0)),4), 'eager', round(e.get('ms_per_step', e.get('p50_ms', 0)),4), 'ms', (d.get('moving_start') or {}).get('p50_ms'))"; }
for c in ${CFGS:-cfg1-demo cfg1 cfg2 cfg4}; do
  for r in 1 2; do run $c 1; run $c 0; done
done
