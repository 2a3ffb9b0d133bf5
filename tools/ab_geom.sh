# A/B on config 3 / config 5 shard (bench.py, device-timed)
b() { timeout 300 env "$@" python bench.py --workload ${WL:-C3} --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('${WL:-C3} $*', round(j['value']), round(j['ms_per_step'],2), j['config']['passes_per_run'], j['gpu_launches'], round(j['roofline']['frac'],3))" ; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_substates.py -x -q -k "eowqs or cluster or gflow or config5 or boundary or shard or loopback or substate" > gpurun_out/pt.log 2>&1; echo pt=$?; tail -1 gpurun_out/pt.log; grep -E "^E |FAILED" gpurun_out/pt.log | head -5
WL=C3E b OWQS_X=1
WL=C3E b OWQS_EOWQS_DECIDE=1
WL=C5E32 b OWQS_X=1
WL=C5E32 b OWQS_EOWQS_DECIDE=1
