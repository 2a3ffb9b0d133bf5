for cfg in "5 2" "6 2" "6 3"; do set -- $cfg
export OWQS_TILE_RB=$1 OWQS_TILE_MINB=$2
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_rb.log 2>&1
tail -1 gpurun_out/b_rb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rb $1 minb $2', round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['per_pass_roofline_frac'],3), d['clocks']['sm_mhz'])"
done
unset OWQS_TILE_RB OWQS_TILE_MINB
timeout 900 python -m pytest tests -q -x -m gpu -k "parity" > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?; tail -1 gpurun_out/pytest_gpu.log
