"""Debug: C1 level, all 22 groups vs the even groups alone - compare bits."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_1705_02003_b200.configs import get
from paper_1705_02003_b200.grouping import device_group
cfg = get("C1")
z = np.load(ROOT / "bench_workloads" / "C1.npz")
solver = cfg.make_solver()
dev = torch.device("cuda", 0)
d_c = torch.from_numpy(z["coords"]).to(dev)
d_k = torch.from_numpy(z["keys"]).to(dev)
n, S = len(z["coords"]), cfg.ensemble_size
groups, pad = device_group(n, S, d_k)
K = pad.numel()
full = solver.run_groups_device(d_c, groups, K, S)
sel = torch.arange(0, K, 2, device=dev)
lanes = groups.view(K, S)[sel].reshape(-1).contiguous()
half = solver.run_groups_device(d_c, lanes, sel.numel(), S)
for name, a, b in zip(["it", "cv", "en", "q"], full, half):
    if name == "en":
        a2 = a[sel]
    else:
        a2 = a.view(K, S)[sel].reshape(-1)
    print(name, torch.equal(a2, b), (a2.double() - b.double()).abs().max().item())
# solve_wave x directly
for G in (K, sel.numel()):
    pass
