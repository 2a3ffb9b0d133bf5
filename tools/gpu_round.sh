timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?
tail -5 gpurun_out/pytest_gpu.log
for w in "C3 128" "C2 128" "C3 64"; do set -- $w
timeout 900 python bench.py --workload $1 --precision $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2.log 2>&1
tail -1 gpurun_out/b_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1 $2', round(d['value']), round(d['ms_per_step'],2), d['config']['passes_per_run'], r and round(r['frac'],3), r and r['bound'], r and round(r['per_pass_roofline_frac'],3))"
done
