nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/sp tools/stream_probe.cu
timeout 300 /tmp/sp
