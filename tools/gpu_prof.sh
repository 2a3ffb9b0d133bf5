for v in OWQS_X=1 OWQS_BFLY4=1; do
env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv python tools/prof_run.py --workload C3 --runs 2 > gpurun_out/ncu_all_$v.csv 2>&1; echo l=$?
done
