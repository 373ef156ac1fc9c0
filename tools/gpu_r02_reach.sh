# frontier / bottom-up reverse reachability: parity tests, then the cfg3 replanning cycle's
# per-kernel split under ncu for each schedule
[ -n "$NOTEST" ] || timeout 900 python -m pytest -x -q tests/test_gpu_query.py tests/test_gpu_replanner.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "query or replanner or reach or relaxed" 2>&1 | tail -4
for v in ${SCHEDS:-grid:64 frontier:64 frontier:8 frontier:0 frontier:256}; do
  impl=${v%%:*}; sw=${v##*:}
  BZG_REACH_IMPL=$impl BZG_REACH_SWITCH=$sw timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rc.csv python tools/replan_cycle.py ${CFG:-cfg3} > gpurun_out/rc_${impl}_$sw.log 2>&1
  python tools/summarize_ncu.py launches gpurun_out/rc.csv gpurun_out/rc_${impl}_$sw.json > /dev/null 2>&1
  rm -f gpurun_out/rc.csv
done
