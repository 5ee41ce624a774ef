#!/bin/bash
# Two concurrent parts with grids small enough for the parts' kernels to be co-resident
# (face SpMV at 2 CTAs/SM, streaming kernels at 1 CTA/SM), C3 level.
run() { echo "== $*"; env "$@" python tools/profile_step.py --config C3 --steps 2 | tail -1; }
run UQG_NONE=1
run UQG_SPMV_B=14
run UQG_SPMV_B=14 UQG_UPDATE_B=7 UQG_DIR_B=7 UQG_FLUSH_B=7
run UQG_SPMV_B=21 UQG_UPDATE_B=7 UQG_DIR_B=7 UQG_FLUSH_B=7
run UQG_UPDATE_B=7 UQG_DIR_B=14 UQG_FLUSH_B=14
run UQG_SOLVE_STREAMS=4 UQG_SPMV_B=14 UQG_UPDATE_B=7 UQG_DIR_B=7 UQG_FLUSH_B=7
