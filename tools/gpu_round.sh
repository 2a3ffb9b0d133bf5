b() { timeout 240 env "$@" python bench.py --workload ${WL:-C3} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('${WL:-C3} $*', round(j['value']), j['ms_per_step'], round(j['roofline']['frac'],3), j['roofline']['bound'])" ; }
b OWQS_X=1
b OWQS_BFLY4=1
WL=C3W b OWQS_X=1
WL=C2 b OWQS_X=1
b OWQS_REMAP=1
b OWQS_TILE_MINB=3
timeout 300 python bench.py --workload C3 --precision 128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
