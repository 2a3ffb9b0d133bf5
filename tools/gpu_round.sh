timeout 1200 python bench.py --workload C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_C4_64.log 2>&1
tail -1 gpurun_out/b_C4_64.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C4 64', round(d['value']), round(d['ms_per_step'],2), d['config']['passes_per_run'], round(r['frac'],3), r['bound'], round(r['per_pass_roofline_frac'],3))"
timeout 1200 python bench.py --workload C3W --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_C3W_64.log 2>&1
tail -1 gpurun_out/b_C3W_64.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C3W 64', round(d['value']), round(d['ms_per_step'],2), d['config']['passes_per_run'], round(r['frac'],3), r['bound'], round(r['per_pass_roofline_frac'],3))"
timeout 1500 python -m pytest tests -q -m gpu -k "sharded or config3 or config5" > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?; tail -1 gpurun_out/pytest_gpu.log
