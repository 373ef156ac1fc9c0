# A/B of the current libbzg against paper_2411_13507_b200/libbzg_v000.so: k_cut_heuristic and
# the step on cfg3 / cfg5-100k (alternating, same box).   gpurun -- bash tools/ab_heur.sh
cd $GRAFT_REPO_ROOT
L=paper_2411_13507_b200
cp $L/libbzg.so $L/libbzg_new.so
run() { python bench.py --config $2 $3 --steps 10 --warmup 3 --no-cpu-baseline --no-planner 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_breakdown_pass']; print('$1', '$2', round(d['ms_per_step'],3), k.get('k_cut_heuristic'), k.get('k_qp_admm'))"; }
for c in "cfg3" "cfg5 --nodes 100000" "cfg2"; do
  run new $c; cp $L/libbzg_v000.so $L/libbzg.so; run old $c; cp $L/libbzg_new.so $L/libbzg.so
  run new $c; cp $L/libbzg_v000.so $L/libbzg.so; run old $c; cp $L/libbzg_new.so $L/libbzg.so
done
rm -f $L/libbzg_new.so
