python tools/pdltest.py
for pdl in 0 1; do
for w in "C2 64" "C2 128" "C3 64"; do set -- $w
if [ $pdl = 0 ]; then export OWQS_NO_PDL=1; else unset OWQS_NO_PDL; fi
timeout 900 python bench.py --workload $1 --precision $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2.log 2>&1
tail -1 gpurun_out/b_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl $1 $2', round(d['value']), round(d['ms_per_step'],3), d['config']['passes_per_run'])"
done; done
unset OWQS_NO_PDL
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?; tail -2 gpurun_out/pytest_gpu.log
