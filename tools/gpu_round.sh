# Round-end evidence on one B200 (run through gpurun from the repo root):
#   GPU tests, smoke, the default bench line, an ncu launch list (time + DRAM bytes + smem bank
#   conflicts per launch) and one `--set full` capture of a heavy tile pass, per-pass times.
# Outputs land in gpurun_out/; copy what is to be judged into profiles/<round>/.
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_default.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/prof_run.py --workload C3 > gpurun_out/ncu_list.log 2>&1; echo list=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:owqs_tile --launch-skip 17 --launch-count 1 -o gpurun_out/full_c3 python tools/prof_run.py --workload C3 > gpurun_out/ncu_full.log 2>&1; echo full=$?
timeout 300 python tools/pass_profile.py --workload C3 --out gpurun_out/passes_c3.json > gpurun_out/pp.log 2>&1; head -1 gpurun_out/pp.log | cut -c1-80
