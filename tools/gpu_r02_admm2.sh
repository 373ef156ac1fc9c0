timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "two_lane" 2>&1 | tail -5
for cfg in cfg2 cfg3; do echo "== $cfg"; CFG=$cfg SPECS="BZG_ADMM_LANES=1;BZG_ADMM_LANES=2" timeout 600 bash tools/ab_env.sh; done
echo "== cfg5 20k"; CFG=cfg5 NODES=20000 SPECS="BZG_ADMM_LANES=1;BZG_ADMM_LANES=2" timeout 600 bash tools/ab_env.sh
