#!/bin/bash
# Round 2, last session: GPU suite, smoke, the driver's two bench arms at the defaults (C3),
# C1 / C2 lines and the ncu launch list of the default bench command.
(time python -m pytest tests -m gpu -x -q) > gpurun_out/r2f2_gputests.log 2>&1; tail -3 gpurun_out/r2f2_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f2_smoke.log 2>&1; tail -1 gpurun_out/r2f2_smoke.log
python bench.py --impl reference > gpurun_out/r2f2_bench_C3_reference_arm.json 2> gpurun_out/r2f2_ref.err
python bench.py > gpurun_out/r2f2_bench_C3.json 2> gpurun_out/r2f2_bench.err
python bench.py --config C2 > gpurun_out/r2f2_bench_C2.json 2>> gpurun_out/r2f2_bench.err
python bench.py --config C1 --steps 20 > gpurun_out/r2f2_bench_C1.json 2>> gpurun_out/r2f2_bench.err
lscpu > gpurun_out/r2f2_lscpu.txt
for f in C3_reference_arm C3 C2 C1; do python -c "
import json,sys
d=json.loads(open('gpurun_out/r2f2_bench_$f.json').read().strip().splitlines()[-1])
print('$f', d.get('value'), (d.get('e2e') or {}).get('value'), d.get('ms_per_step'), (d.get('parity') or {}).get('ok'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('reasons'))"; done
