set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/mp tools/march_probe.cu
timeout 600 /tmp/mp 512 32 42 16 > gpurun_out/march_c3.log 2>&1; echo mp=$?
cat gpurun_out/march_c3.log
timeout 300 /tmp/mp 256 16 93 8 > gpurun_out/march_c2.log 2>&1; echo mp2=$?
cat gpurun_out/march_c2.log
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "kl or smoke or fem3d_kl or anisotropy" 2>&1 | tail -3
python tools/profile_step.py --config C5 --maxit 4 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"kl_sep2d" -c 2 python tools/profile_step.py --config C5 --maxit 4 > gpurun_out/ncu_kl2.log 2>&1; grep -E "kl_sep|duration|bytes|pct" gpurun_out/ncu_kl2.log | head -20
