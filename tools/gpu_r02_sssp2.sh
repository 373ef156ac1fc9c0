timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k live_reference -s 2>&1 | grep -v "^$" | tail -25
for b in 1 2 4; do echo "== blocks/SM $b"; BZG_BF_BLOCKS_PER_SM=$b python tools/sssp_probe.py cfg3 3; BZG_BF_BLOCKS_PER_SM=$b python tools/sssp_probe.py cfg5:100000 3; done 2>&1 | cut -c1-120
