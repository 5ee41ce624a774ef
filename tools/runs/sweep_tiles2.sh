run() { python tools/profile_step.py --config $1 --steps 2 2>&1 | tail -2; }
U4="-DUQG_UPDATE_TILES=4 -DUQG_UPDATE_MINB=2"
for v in "$U4 -DUQG_DIR_TILES=4 -DUQG_DIR_MINB=2" "$U4 -DUQG_DIR_TILES=4 -DUQG_DIR_MINB=2 -DUQG_DIR_FLAT=1" "$U4 -DUQG_DIR_TILES=8 -DUQG_DIR_MINB=1 -DUQG_DIR_FLAT=1" "$U4 -DUQG_DIR_TILES=2 -DUQG_DIR_FLAT=1" "$U4 -DUQG_DIR_TILES=4 -DUQG_DIR_MINB=2 -DUQG_UPDATE_BATCH=8"; do
  UQG_NVCC_EXTRA="$v" python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
  echo "== $v"; run C3; run C2
done
