# A/B of the current libbzg against paper_2411_13507_b200/libbzg_v000.so on the build kernels
# (k_expand, k_pair_list) and the step (alternating, same box).   gpurun -- bash tools/ab_build.sh
cd $GRAFT_REPO_ROOT
L=paper_2411_13507_b200
cp $L/libbzg.so $L/libbzg_new.so
run() { python bench.py $2 --steps 10 --warmup 3 --no-cpu-baseline --no-planner 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_breakdown_pass']; print('$1', '$2', round(d['ms_per_step'],3), k.get('k_expand'), k.get('k_pair_list'))"; }
for c in "--config cfg3" "--config cfg2" "--config cfg5 --nodes 100000"; do
  run new "$c"; cp $L/libbzg_v000.so $L/libbzg.so; run old "$c"; cp $L/libbzg_new.so $L/libbzg.so
  run new "$c"; cp $L/libbzg_v000.so $L/libbzg.so; run old "$c"; cp $L/libbzg_new.so $L/libbzg.so
done
rm -f $L/libbzg_new.so
