python tools/profile_step.py --config C1 --steps 2 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pcg_cluster_smem|pcg_persistent" -c 1 -o gpurun_out/r02_prof_c1_smem python tools/profile_step.py --config C1 > gpurun_out/ncu_c1_smem.log 2>&1; echo ncu=$?
UQG_PCG_PERSISTENT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pcg_cluster_smem|pcg_persistent" -c 1 -o gpurun_out/r02_prof_c1_cl python tools/profile_step.py --config C1 > gpurun_out/ncu_c1_cl.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_c1_smem.log
