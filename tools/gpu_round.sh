set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/b_c3_jit.log 2>&1; echo b1=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --flags 128 > gpurun_out/b_c3_aot.log 2>&1; echo b2=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?
tail -3 gpurun_out/pytest_gpu.log
