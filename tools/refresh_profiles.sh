# Refresh the round's bench lines, the cfg3 launch list, the cfg3 `ncu --set full` capture and the
# row-block table on a GPU box (one GPU):   gpurun --timeout 3600 -- 'R=r02 bash tools/refresh_profiles.sh'
# (the ncu summaries are written on the box: gpurun_out/${R}_ncu_full_cfg3.json, ${R}_launches_cfg3.json)
cd "${GRAFT_REPO_ROOT:-.}"
R=${R:-r02}
mkdir -p gpurun_out
for c in cfg1 cfg1-demo cfg2 cfg3 cfg4; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${R}_bench_$c.json 2> gpurun_out/err_$c.txt
done
for n in 10000 20000 50000 100000; do
  python bench.py --config cfg5 --nodes $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_bench_cfg5_$n.json 2> gpurun_out/err_cfg5_$n.txt
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_reference_arm_cfg3.json 2>&1
python tools/row_block_probe.py cfg3 5 > gpurun_out/${R}_row_blocks_cfg3.jsonl 2> gpurun_out/err_rbp.txt
# replanning cycles (eager vs captured) and the launch list of captured cfg1-demo / cfg2 cycles
python tools/replan_probe.py cfg1-demo cfg2 cfg3 > gpurun_out/${R}_replan_cycles.jsonl 2> gpurun_out/err_replan.txt
for c in cfg1-demo cfg2; do
  python tools/replan_cycle.py $c 3 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/replan_launches_$c.csv \
      python tools/replan_cycle.py $c 3 > /dev/null 2>&1
done
# launch list of the same bench command (cold-cache, serialised: compare shares, not times)
python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
# full capture of the hot kernels of one cfg3 step
python tools/run_once.py cfg3 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k 'regex:k_qp_admm|k_cut_heuristic|k_pair_list|k_qp_polish|k_bf_scan|k_expand' -c 6 -f \
    -o /tmp/prof_${R}_full python tools/run_once.py cfg3 1 > gpurun_out/ncu_full.log 2>&1
# summaries on the box (the report itself exceeds what gpurun copies back)
python tools/summarize_ncu.py full /tmp/prof_${R}_full.ncu-rep gpurun_out/${R}_ncu_full_cfg3.json > /dev/null 2>&1
python tools/summarize_ncu.py launches gpurun_out/launches.csv gpurun_out/${R}_launches_cfg3.json > /dev/null 2>&1
for c in cfg1-demo cfg2; do
  python tools/summarize_ncu.py launches gpurun_out/replan_launches_$c.csv gpurun_out/${R}_replan_launches_$c.json > /dev/null 2>&1
done
echo done
