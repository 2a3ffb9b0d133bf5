nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/membench tools/membench.cu && /tmp/membench > gpurun_out/membench.log 2>&1
cat gpurun_out/membench.log
