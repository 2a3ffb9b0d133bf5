# alternating A/B repeats on config 3 (bench.py, device-timed)
b() { timeout 300 env "$@" python bench.py --workload ${WL:-C3} --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('${WL:-C3} $*', round(j['value']), round(j['ms_per_step'],2))" ; }
for r in 1 2 3; do b OWQS_X=1; b OWQS_BEAM=16 OWQS_EXPAND=12; done
WL=C3W b OWQS_X=1; WL=C3W b OWQS_BEAM=16 OWQS_EXPAND=12
