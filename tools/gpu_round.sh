timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo b=$?
tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('def', round(d['value']), round(d['ms_per_step'],2), d['e2e'], d['roofline']['frac'], d['roofline']['per_pass_roofline_frac'])"
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?; tail -1 gpurun_out/pytest_gpu.log
