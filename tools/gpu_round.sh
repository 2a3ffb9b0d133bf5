for rb in 5 6; do
OWQS_TILE_RB=$rb timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/b_rb$rb.log 2>&1
tail -1 gpurun_out/b_rb$rb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rb $rb', round(d['value']), d['ms_per_step'], d['config']['passes_per_run'], round(d['roofline']['per_pass_roofline_frac'],3), d['clocks']['sm_mhz'])"
done
OWQS_TILE_RB=6 timeout 300 python tools/pass_profile.py --workload C3 --out gpurun_out/pp_c3_rb6.json > gpurun_out/pp_rb6.log 2>&1
OWQS_TILE_RB=5 timeout 300 python tools/pass_profile.py --workload C3 --out gpurun_out/pp_c3_rb5.json > gpurun_out/pp_rb5.log 2>&1
OWQS_TILE_RB=6 timeout 900 python -m pytest tests -x -q -m gpu -k "parity" > gpurun_out/pytest_rb6.log 2>&1; echo pt=$?; tail -2 gpurun_out/pytest_rb6.log
