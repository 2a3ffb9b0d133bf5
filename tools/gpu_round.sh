# A/B: tile occupancy (2 vs 3 CTAs/SM), RB 5 vs 6, remapping; quick parity subset under each
b() { timeout 240 env "$@" python bench.py --workload C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.readlines()[-1]); print('$*', round(j['value']), j['ms_per_step'], j['roofline']['frac'])" ; }
b OWQS_X=0
b OWQS_TILE_MINB=3
b OWQS_REMAP=1
b OWQS_REMAP=1 OWQS_TILE_MINB=3
b OWQS_TILE_RB=6
b OWQS_TILE_RB=6 OWQS_REMAP=1
b OWQS_TILE_RB=6 OWQS_TILE_MINB=2
OWQS_TILE_MINB=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not inner" > gpurun_out/pt3.log 2>&1; echo pt3=$?; tail -1 gpurun_out/pt3.log
OWQS_TILE_RB=6 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not inner" > gpurun_out/pt6.log 2>&1; echo pt6=$?; tail -1 gpurun_out/pt6.log
