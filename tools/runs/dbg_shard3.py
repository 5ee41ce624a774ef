"""Debug: does a C1 solve depend on what ran before in the process?"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_1705_02003_b200.configs import get
from paper_1705_02003_b200.grouping import device_group
order = sys.argv[1]  # e.g. "half,full" or "full,half"
cfg = get("C1")
z = np.load(ROOT / "bench_workloads" / "C1.npz")
solver = cfg.make_solver()
dev = torch.device("cuda", 0)
d_c = torch.from_numpy(z["coords"]).to(dev)
d_k = torch.from_numpy(z["keys"]).to(dev)
n, S = len(z["coords"]), cfg.ensemble_size
groups, pad = device_group(n, S, d_k)
K = pad.numel()
sel = torch.arange(0, K, 2, device=dev)
out = {}
for what in order.split(","):
    if what == "full":
        it, cv, en, q = solver.run_groups_device(d_c, groups, K, S)
        out[what] = q.view(K, S)[sel].cpu().numpy()
    else:
        lanes = groups.view(K, S)[sel].reshape(-1).contiguous()
        it, cv, en, q = solver.run_groups_device(d_c, lanes, sel.numel(), S)
        out[what] = q.view(-1, S).cpu().numpy()
    np.save(f"/tmp/q_{order.replace(',', '_')}_{what}.npy", out[what])
print(order, {k: float(v[0, 0]) for k, v in out.items()})
