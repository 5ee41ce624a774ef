# build-knob / env sweep on C3 (and C2): step times only (not bench values)
set -x
run() { python tools/profile_step.py --config $1 --steps 3 2>&1 | tail -3; }
python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
echo "== base"; run C3; run C2
echo "== defer8"; UQG_X_DEFER=8 run C3; UQG_X_DEFER=8 run C2
for h in 1 2; do
  UQG_NVCC_EXTRA="-DUQG_FACE_HINT=$h" python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
  echo "== hint$h"; run C3; run C2
  echo "== hint$h defer8"; UQG_X_DEFER=8 run C3
done
