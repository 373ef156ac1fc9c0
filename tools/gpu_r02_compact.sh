timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "schedules or cut_and_path" 2>&1 | tail -4
for cfg in cfg2 cfg3; do echo "== $cfg"; CFG=$cfg SPECS="BZG_ADMM_PASSES=1;BZG_ADMM_PASSES=3;BZG_ADMM_PASSES=3 BZG_ADMM_DUMP=20;BZG_ADMM_PASSES=4 BZG_ADMM_DUMP=6" timeout 900 bash tools/ab_env.sh; done
echo "== cfg5 20k"; CFG=cfg5 NODES=20000 SPECS="BZG_ADMM_PASSES=1;BZG_ADMM_PASSES=3;BZG_ADMM_PASSES=3 BZG_ADMM_DUMP=20" timeout 600 bash tools/ab_env.sh
