#!/bin/bash
# ncu DRAM bytes and durations of the four PCG kernels at C4 and C5 (throughput mode: 48
# iterations per group, one stream so a launch covers every group): the traffic behind the
# C4 / C5 fractions.  (A --set full capture of 16 such launches took 21 minutes and its
# reports exceeded the 64 MiB return limit; the three metrics below are what is needed.)
for c in C4 C5; do
  UQG_SOLVE_STREAMS=1 python tools/profile_step.py --config $c --maxit 48 | tail -1
  UQG_SOLVE_STREAMS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"pcg_(spmv_fv2d|update|dir|flush)" -s 36 -c 32 --csv \
    --log-file gpurun_out/r2m_launches_$c.csv python tools/profile_step.py --config $c --maxit 48 \
    > gpurun_out/r2m_ncu_$c.log 2>&1
  tail -1 gpurun_out/r2m_ncu_$c.log
done
