# A/B of the current libbzg against paper_2411_13507_b200/libbzg_v000.so on cfg3 and cfg2
# (alternating, same box).   gpurun -- bash tools/ab_admm.sh
cd $GRAFT_REPO_ROOT
L=paper_2411_13507_b200
cp $L/libbzg.so $L/libbzg_new.so
run() { python bench.py --config $2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_breakdown_pass']; print('$1', '$2', round(d['ms_per_step'],3), k['k_qp_admm'], round(d['roofline']['frac'],3))"; }
for c in cfg3 cfg2; do
  run new $c; cp $L/libbzg_v000.so $L/libbzg.so; run old $c; cp $L/libbzg_new.so $L/libbzg.so
  run new $c; cp $L/libbzg_v000.so $L/libbzg.so; run old $c; cp $L/libbzg_new.so $L/libbzg.so
done
