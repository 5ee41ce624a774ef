set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/lscpu.txt
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gputests.log 2>&1; echo tests_rc=$?
tail -8 gpurun_out/r02_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/r02_bench_C3.json 2> gpurun_out/r02_bench_C3.err; echo bench_rc=$?
tail -c 4000 gpurun_out/r02_bench_C3.json
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02_bench_C3_ref.json 2> gpurun_out/r02_bench_C3_ref.err; echo ref_rc=$?
tail -c 2000 gpurun_out/r02_bench_C3_ref.json
python bench.py --config C1 --steps 20 --warmup 5 > gpurun_out/r02_bench_C1.json 2> gpurun_out/r02_bench_C1.err; echo bench1_rc=$?
tail -c 2500 gpurun_out/r02_bench_C1.json
