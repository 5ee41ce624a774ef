set -x
python tools/runs/dbg_shard.py
UQG_PCG_PERSISTENT=0 python tools/runs/dbg_shard.py
UQG_PCG_PERSISTENT=1 python tools/runs/dbg_shard.py
python -m pytest tests -m gpu -v -p no:cacheprovider > gpurun_out/r02_gputests_v.log 2>&1; echo rc=$?
tail -40 gpurun_out/r02_gputests_v.log
