#!/bin/bash
# Second grid sweep at C3 (single stream): more blocks for dir / flush, and the update /
# face SpMV kernels off their residency-sized grids.
run() {
  echo "== $*"
  env UQG_SOLVE_STREAMS=1 "$@" python bench.py --steps 1 --warmup 1 --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], {k:(round(v['ms'],1), round(v['frac'],3)) for k,v in d['roofline']['pcg_kernels'].items()})"
}
run UQG_DIR_B=170 UQG_FLUSH_B=170 UQG_UPDATE_B=14 UQG_SPMV_B=28
run UQG_DIR_B=256 UQG_FLUSH_B=256 UQG_UPDATE_B=28 UQG_SPMV_B=42
run UQG_DIR_B=511 UQG_FLUSH_B=511 UQG_UPDATE_B=56 UQG_SPMV_B=56
run UQG_DIR_B=112 UQG_FLUSH_B=112 UQG_UPDATE_B=112 UQG_SPMV_B=63
