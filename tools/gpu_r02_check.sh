# round-2 GPU check: full gpu test suite + short benches (cfg3, cfg2) with per-kernel breakdown
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1 | tail -25 > gpurun_out/r02_pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 --breakdown --no-cpu-baseline > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --breakdown --no-cpu-baseline > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err
tail -3 gpurun_out/r02_pytest_gpu.txt
