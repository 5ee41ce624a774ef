set -x
python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
python -m pytest tests/test_gpu_report.py -q -x -p no:cacheprovider 2>&1 | tail -15
run() { python tools/profile_step.py --config $1 --steps 3 2>&1 | tail -3; }
echo "== base"; run C3; run C2
for v in "-DUQG_FACE_PF=1" "-DUQG_FACE_PF=1 -DUQG_FACE_MINB=3"; do
  UQG_NVCC_EXTRA="$v" python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
  echo "== $v"; run C3; run C2
done
