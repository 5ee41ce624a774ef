nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/csp tools/cluster_sync_probe.cu
for m in 0 1 2 3; do timeout 120 /tmp/csp $m; done
