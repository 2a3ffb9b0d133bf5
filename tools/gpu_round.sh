OWQS_T0_FREE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_determinism.py -x -q -k "not config4" > gpurun_out/pt.log 2>&1; echo pt=$?; tail -1 gpurun_out/pt.log; grep -E "^E |FAILED" gpurun_out/pt.log | head -5
b() { timeout 240 env "$@" python bench.py --workload ${WL:-C3} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('${WL:-C3} $*', round(j['value']), j['ms_per_step'], round(j['roofline']['frac'],3))" ; }
b OWQS_X=1
b OWQS_T0_FREE=1
WL=C3W b OWQS_X=1
WL=C3W b OWQS_T0_FREE=1
