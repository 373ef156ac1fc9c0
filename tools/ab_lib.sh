# Same-box A/B of two builds of libbzg: the current build vs paper_2411_13507_b200/libbzg_v000.so
# (built by hand with the variant flags), alternating twice.  CFG=cfg3 by default.
#   gpurun -- bash tools/ab_lib.sh
cd $GRAFT_REPO_ROOT
L=paper_2411_13507_b200
cp $L/libbzg.so $L/libbzg_new.so
run() { python bench.py --config ${CFG:-cfg3} ${NODES:+--nodes $NODES} --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3), d['kernels_ms_breakdown_pass']['k_qp_admm'], d['kernels_ms_breakdown_pass'].get('k_cut_heuristic'), d['kernels_ms_breakdown_pass'].get('k_expand'))"; }
run new; cp $L/libbzg_v000.so $L/libbzg.so; run old; cp $L/libbzg_new.so $L/libbzg.so; run new; cp $L/libbzg_v000.so $L/libbzg.so; run old
cp $L/libbzg_new.so $L/libbzg.so
