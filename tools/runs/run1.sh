set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_C3_a.json 2> gpurun_out/r02_bench_C3_a.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r02_bench_C3_a.json
python bench.py --config C1 --steps 20 --warmup 5 > gpurun_out/r02_bench_C1_a.json 2> gpurun_out/r02_bench_C1_a.err; echo bench1_rc=$?
