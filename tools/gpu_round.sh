timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_async.py -x -q -k "not config4" > gpurun_out/pt.log 2>&1; echo pt=$?; tail -1 gpurun_out/pt.log; grep -E "^E " gpurun_out/pt.log | head -5
b() { timeout 240 env "$@" python bench.py --workload ${WL:-C3} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('${WL:-C3} $*', round(j['value']), j['ms_per_step'], round(j['roofline']['frac'],3), j['roofline']['bound'])" ; }
b OWQS_X=1
b OWQS_NO_BANKCLS=1
WL=C3W b OWQS_X=1
WL=C3E b OWQS_X=1
timeout 900 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum --clock-control none --csv -k regex:owqs_tma python tools/prof_run.py --workload C3 > gpurun_out/ncu_bank2.csv 2>&1; echo ncu=$?
