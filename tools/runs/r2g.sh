for m in 2 3; do UQG_PCG_PERSISTENT=$m timeout 300 python tools/persistent_probe.py 2>&1 | tail -7; done
timeout 300 python -m pytest tests/test_gpu_persistent.py -q -x -p no:cacheprovider -k bitwise 2>&1 | tail -2
