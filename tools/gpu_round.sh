b() { timeout 240 env "$@" python bench.py --workload ${WL:-C3} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('${WL:-C3} $*', round(j['value']), j['ms_per_step'], j['config']['passes_per_run'])" ; }
b OWQS_X=1
b OWQS_KWIDE=6
b OWQS_KWIDE=5
b OWQS_REMAP_MARGIN=0
b OWQS_REMAP_MARGIN=2
b OWQS_REMAP_MARGIN=4
