nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/mp tools/march_probe.cu
timeout 600 /tmp/mp 512 32 42 16 > gpurun_out/march2_c3.log 2>&1; echo mp=$?
cat gpurun_out/march2_c3.log
timeout 300 /tmp/mp 256 16 93 8 > gpurun_out/march2_c2.log 2>&1; echo mp2=$?
cat gpurun_out/march2_c2.log
