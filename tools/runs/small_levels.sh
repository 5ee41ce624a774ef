#!/bin/bash
# Per-rank work of the strong-scaling step at N = 2, 4, 8 emulated on one GPU: the first
# 21 / 11 / 6 groups of the C3 level (time per group-iteration vs the full 42-group level).
for ns in 1328 672 352 192; do
  echo "== max-samples $ns"
  python bench.py --max-samples $ns --steps 2 --warmup 1 --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
gi=d['pcg_loop']['group_iterations']/d['steps'] if 'pcg_loop' in d else None
print(d['value'], d['ms_per_step'], 'group-iters/step', gi, 'us per group-iteration', None if not gi else 1e3*d['ms_per_step']/gi, {k:round(v['frac'],3) for k,v in d['roofline']['pcg_kernels'].items()})"
done
