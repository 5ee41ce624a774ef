set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r2b_gputests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r2b_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
python tools/profile_step.py --config C5 --maxit 4 > gpurun_out/plain_c5.log 2>&1; echo plain_c5=$?
tail -3 gpurun_out/plain_c5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kl_sep2d|kl_tile|assemble_fv2d_faces" -c 3 -o gpurun_out/r02_prof_klasm_C5 python tools/profile_step.py --config C5 --maxit 4 > gpurun_out/ncu_c5.log 2>&1; echo ncu_c5=$?
tail -5 gpurun_out/ncu_c5.log
