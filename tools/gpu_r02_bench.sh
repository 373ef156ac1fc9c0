# bench lines (cfg3 default with cpu_baseline, cfg2, cfg1, cfg4, cfg5) + the reference arm for cfg3
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err; tail -c 3000 gpurun_out/r02_bench_cfg3.json
for c in cfg1 cfg2 cfg4; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_$c.json 2>/dev/null; done
for n in 10000 100000; do python bench.py --config cfg5 --nodes $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_cfg5_$n.json 2>/dev/null; done
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_arm_cfg3.json 2>&1; tail -c 1500 gpurun_out/r02_bench_reference_arm_cfg3.json
