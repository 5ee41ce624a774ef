set -x
python -m pytest tests -m gpu -x -q -k "scale_parity or ref_conformance or gpu_dist or group" 2>&1 | tail -15
python -m pytest tests -m gpu -q -rs 2>&1 | tail -8
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_C3_b.json 2> gpurun_out/r02_bench_C3_b.err; echo bench_rc=$?
export UQG_SOLVE_STREAMS=1
python tools/profile_step.py --config C3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pcg_(spmv_fv2d|update|dir|flush)" -s 400 -c 13 -o gpurun_out/r02_prof_pcg_C3 python tools/profile_step.py --config C3 > gpurun_out/ncu_c3.log 2>&1; echo ncu_c3=$?
python tools/profile_step.py --config C5 --maxit 4 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"kl_sep2d|assemble_fv2d_faces" -c 2 -o gpurun_out/r02_prof_klasm_C5 python tools/profile_step.py --config C5 --maxit 4 > gpurun_out/ncu_c5.log 2>&1; echo ncu_c5=$?
