# A/B of tile geometries on config 3 (bench.py, device-timed)
b() { timeout 300 env "$@" python bench.py --workload ${WL:-C3} --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('${WL:-C3} $*', round(j['value']), round(j['ms_per_step'],2), j['config']['passes_per_run'], round(j['roofline']['frac'],3))" ; }
b OWQS_X=1
b OWQS_TILE_RB=6
b OWQS_TILE_RB=6 OWQS_TILE_MINB=6
b OWQS_TILE_RB=6 OWQS_TILE_MINB=8
