timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python tools/sssp_probe.py cfg3
python tools/sssp_probe.py cfg2
python tools/sssp_probe.py cfg5:100000
BZG_TRACE=1 python tools/run_once.py cfg3 2>&1 | grep "bzg path"
