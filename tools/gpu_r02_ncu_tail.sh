export BZG_ADMM_PASSES=2 BZG_ADMM_DUMP=12
python tools/run_once.py cfg2 > gpurun_out/plain_tail.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_qp_admm -c 2 \
   -o gpurun_out/r02_admm_tail_cfg2 python tools/run_once.py cfg2 > gpurun_out/ncu_tail.log 2>&1
ls -la gpurun_out/r02_admm_tail_cfg2.ncu-rep
