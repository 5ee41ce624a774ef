run() { python tools/profile_step.py --config $1 --steps 2 2>&1 | tail -2; }
python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
echo "== base"; run C3
for v in "-DUQG_UPDATE_TILES=4 -DUQG_UPDATE_MINB=2 -DUQG_DIR_TILES=4 -DUQG_DIR_MINB=2" "-DUQG_UPDATE_TILES=3 -DUQG_UPDATE_MINB=2 -DUQG_DIR_TILES=3 -DUQG_DIR_MINB=2" "-DUQG_DIR_TILES=4 -DUQG_DIR_MINB=2" "-DUQG_UPDATE_TILES=4 -DUQG_UPDATE_MINB=2"; do
  UQG_NVCC_EXTRA="$v" python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
  echo "== $v"; run C3
done
