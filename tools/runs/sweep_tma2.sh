run() { python tools/profile_step.py --config $1 --steps 2 2>&1 | tail -2; }
python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
echo "== base"; run C3
UQG_NVCC_EXTRA="-DUQG_FACE_BATCH=4" python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
for n in 1 2; do echo "== batch4 tma$n"; UQG_FACE_TMA=$n run C3; done
UQG_NVCC_EXTRA="-DUQG_FACE_BATCH=2" python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
for n in 1 2; do echo "== batch2 tma$n"; UQG_FACE_TMA=$n run C3; done
