timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo b=$?
tail -1 gpurun_out/bench_default.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3_tile.csv python tools/prof_run.py --workload C3 > gpurun_out/ncu_ll.log 2>&1; echo ll=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:owqs_tma_c64 --launch-skip 20 --launch-count 1 -o gpurun_out/ncu_tile_c3_p20 python tools/prof_run.py --workload C3 > gpurun_out/ncu_t.log 2>&1; echo t=$?
