"""Lock-step diagnostic: solve every golden level's plan with the device solver
and report iteration / QoI differences against the reference golden study.

    python tools/diag_study.py pde_test1
"""

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1705_02003_b200 as uq  # noqa: E402
from paper_1705_02003_b200.grouping import GroupingPlan  # noqa: E402


def main(name):
    gold = json.loads((ROOT / "tests" / "golden" / f"{name}_study.json").read_text())
    cfg = uq.PRESETS_3D.get(name) or uq.CONFIGS[name]
    solver = cfg.make_solver()
    for lv in gold["levels"]:
        plan = GroupingPlan(lv["level"], cfg.ensemble_size, tuple(tuple(g) for g in lv["ensembles"]),
                            tuple(lv["padding"]), "sur")
        coords = {sid: np.array(c) for sid, c in zip(lv["ids"], lv["coords"])}
        iters, qois, _ = solver.solve_plan(plan, coords)
        d_it = [iters[s] - i for s, i in zip(lv["ids"], lv["iterations"])]
        d_q = [abs(qois[s] - q) / abs(q) for s, q in zip(lv["ids"], lv["qoi"])]
        bad = [(s, iters[s], i) for s, i in zip(lv["ids"], lv["iterations"]) if iters[s] != i]
        print(f"level {lv['level']}: {len(lv['ids'])} samples, max|d_it|={max(map(abs, d_it))}, "
              f"n_it_diff={sum(1 for x in d_it if x)}, max rel dQoI={max(d_q):.2e}, diffs={bad[:8]}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "pde_test1")
