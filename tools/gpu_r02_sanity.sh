set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02_pytest_gpu_a.txt
timeout 600 compute-sanitizer --tool memcheck --leak-check no python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_memcheck_smoke.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/run_once.py cfg1 > gpurun_out/r02_memcheck_cfg1.txt 2>&1
tail -5 gpurun_out/r02_pytest_gpu_a.txt gpurun_out/r02_memcheck_smoke.txt gpurun_out/r02_memcheck_cfg1.txt
