python tools/runs/dbg_shard3.py half
python tools/runs/dbg_shard3.py full
python tools/runs/dbg_shard3.py half,full
python tools/runs/dbg_shard3.py full,half
UQG_PCG_PERSISTENT=0 python tools/runs/dbg_shard3.py half
UQG_PCG_PERSISTENT=0 python tools/runs/dbg_shard3.py full
