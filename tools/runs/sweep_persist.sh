for v in "" "-DUQG_PERSIST_ROWS=1" "-DUQG_PERSIST_ROWS=1 -DUQG_PERSIST_MINB=3"; do
  UQG_NVCC_EXTRA="$v" python -c "from paper_1705_02003_b200 import build as b; b.build(force=True)"
  echo "== $v"; UQG_PCG_PERSISTENT=2 timeout 300 python tools/persistent_probe.py 2>&1 | grep -E "K= 4|K= 7|K=22"
  timeout 300 python -m pytest tests/test_gpu_persistent.py -q -x -p no:cacheprovider -k bitwise 2>&1 | tail -1
done
