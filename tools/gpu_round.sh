timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?
tail -15 gpurun_out/pytest_gpu.log | cut -c1-300
timeout 300 python tools/pass_profile.py --workload C3 --out gpurun_out/pp_c3_e3.json > gpurun_out/pp_c3_e3.log 2>&1; echo pp=$?
head -1 gpurun_out/pp_c3_e3.log | cut -c1-100
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_c3_e3.log 2>&1; echo b1=$?
tail -1 gpurun_out/b_c3_e3.log | cut -c1-200
