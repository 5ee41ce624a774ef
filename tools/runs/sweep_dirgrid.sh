#!/bin/bash
# Blocks per group of pcg_dir / pcg_flush at C3 (single stream: one launch covers all 42
# groups; 2 CTAs/SM -> 296 resident blocks).  Per-kernel times from the bench's profiled pass.
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp tools/stream_probe.cu && /tmp/sp > gpurun_out/s5i_stream_probe.txt 2>&1
tail -20 gpurun_out/s5i_stream_probe.txt
for b in 0 7 14 21 28 56 63 112; do
  echo "== UQG_DIR_B=$b UQG_FLUSH_B=$b"
  UQG_SOLVE_STREAMS=1 UQG_DIR_B=$b UQG_FLUSH_B=$b python bench.py --steps 1 --warmup 1 --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], {k:(round(v['ms'],1), round(v['frac'],3)) for k,v in d['roofline']['pcg_kernels'].items()})"
done
