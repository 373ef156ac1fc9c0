# ncu --set full of k_qp_admm on cfg2, one lane vs two lanes per instance
for L in 1 2; do
  BZG_ADMM_LANES=$L python tools/run_once.py cfg2 > gpurun_out/plain_l$L.log 2>&1 && \
  BZG_ADMM_LANES=$L ncu --set full --clock-control none --import-source on -k regex:k_qp_admm -c 1 \
     -o gpurun_out/r02_admm_cfg2_l$L python tools/run_once.py cfg2 > gpurun_out/ncu_l$L.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
