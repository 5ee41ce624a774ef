set -x
UQG_FACE_TMA=2 timeout 900 python -m pytest tests/test_gpu_faces.py -q -x -p no:cacheprovider 2>&1 | tail -3
run() { python tools/profile_step.py --config $1 --steps 3 2>&1 | tail -3; }
echo "== base"; run C3; run C2
for n in 2 3 4; do echo "== tma$n"; UQG_FACE_TMA=$n run C3; UQG_FACE_TMA=$n run C2; done
