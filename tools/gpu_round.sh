for w in "C3 64" "C3 128" "C2 64"; do set -- $w
timeout 900 python bench.py --workload $1 --precision $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2.log 2>&1
tail -1 gpurun_out/b_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['ms_per_step'],3), d['config']['passes_per_run'], d['gpu_launches'])"
done
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?; tail -1 gpurun_out/pytest_gpu.log
