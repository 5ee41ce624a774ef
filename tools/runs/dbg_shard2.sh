set -x
cd $GRAFT_REPO_ROOT
export UQG_BENCH_SHARE_GPU=1
for mode in 2 0 1; do
 for rep in a b; do
  UQG_PCG_PERSISTENT=$mode python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_level.py --config C1 --out /tmp/lvl_${mode}_${rep}.json > /dev/null 2>&1
 done
 UQG_PCG_PERSISTENT=$mode python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 tools/dist_level.py --config C1 --out /tmp/lvl_${mode}_one.json > /dev/null 2>&1
done
python - <<'PY'
import json
for mode in "201":
    a=json.load(open(f"/tmp/lvl_{mode}_a.json")); b=json.load(open(f"/tmp/lvl_{mode}_b.json")); o=json.load(open(f"/tmp/lvl_{mode}_one.json"))
    def d(x,y): return max(abs(u-v) for u,v in zip(x["qoi"],y["qoi"]))
    print(mode, "a-b", d(a,b), "a-one", d(a,o), "b-one", d(b,o), "iters eq", a["iters"]==o["iters"])
    print("  first diffs", [i for i,(u,v) in enumerate(zip(a["qoi"],o["qoi"])) if u!=v][:20])
PY
