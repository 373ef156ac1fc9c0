# Same-box A/B of environment knobs on one build: each "VAR=val ..." spec in $SPECS runs bench.py
# (CFG, default cfg3) twice, interleaved.   gpurun -- 'SPECS="A=1;A=0" bash tools/ab_env.sh'
cd "${GRAFT_REPO_ROOT:-.}"
IFS=';' read -ra S <<< "$SPECS"
for rep in 1 2; do
  for spec in "${S[@]}"; do
    env $spec python bench.py --config ${CFG:-cfg3} ${NODES:+--nodes $NODES} --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['ms_per_step'],3), d['kernels_ms_breakdown_pass']['k_qp_admm'])"
  done
done
