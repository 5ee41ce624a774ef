# face SpMV occupancy / batch variants (same bits): per-kernel ms at C2 and C3
set -x
for v in "" "-DUQG_FACE_MINB=5 -DUQG_FACE_BATCH=4" "-DUQG_FACE_MINB=4 -DUQG_FACE_BATCH=4" "-DUQG_FACE_MINB=6 -DUQG_FACE_BATCH=2"; do
  UQG_NVCC_EXTRA="$v" python -c "import sys; sys.path.insert(0,'.'); from paper_1705_02003_b200 import build as b; b.build(force=True)" || continue
  tag=$(echo "$v" | tr -d ' =-' )
  python bench.py --config C2 --steps 3 --warmup 3 --prof-steps 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_C2_${tag}.json 2>/dev/null
  python bench.py --config C3 --steps 2 --warmup 3 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_C3_${tag}.json 2>/dev/null
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1705_02003_b200 import build as b; b.build(force=True)"
UQG_X_DEFER=8 python bench.py --config C2 --steps 3 --warmup 3 --prof-steps 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_C2_kx8.json 2>/dev/null
UQG_X_DEFER=8 python bench.py --config C3 --steps 2 --warmup 3 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_C3_kx8.json 2>/dev/null
