for rep in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_fin.log 2>&1
tail -1 gpurun_out/b_fin.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fin', round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['per_pass_roofline_frac'],3), d['clocks']['sm_mhz'], d['gpu_launches'])"
done
timeout 300 python tools/pass_profile.py --workload C3 --out gpurun_out/pp_c3_fin.json > gpurun_out/pp_fin.log 2>&1; head -1 gpurun_out/pp_fin.log | cut -c1-80
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?; tail -1 gpurun_out/pytest_gpu.log
