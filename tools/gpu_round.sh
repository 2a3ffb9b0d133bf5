timeout 1500 python -m pytest tests -q -m gpu -k "standard_form or random_patterns" > gpurun_out/pytest_gpu.log 2>&1; echo pt=$?; tail -3 gpurun_out/pytest_gpu.log
