#!/bin/bash
# pcg_dir traversal: chunk-strided (library) vs flat tile-strided, blocks per group, C3.
run() {
  echo "== $*"
  env UQG_SOLVE_STREAMS=1 "$@" python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], {k:(round(v['ms'],1), round(v['frac'],3)) for k,v in d['roofline']['pcg_kernels'].items()}, d['parity']['ok'])"
}
run UQG_DIR_FLAT=0
run UQG_DIR_FLAT=1 UQG_DIR_B=7
run UQG_DIR_FLAT=1 UQG_DIR_B=14
run UQG_DIR_FLAT=1
run UQG_DIR_FLAT=1 UQG_DIR_B=112
echo default two-part mode
for f in 0 1; do UQG_DIR_FLAT=$f python tools/profile_step.py --config C3 --steps 2 | tail -1; done
