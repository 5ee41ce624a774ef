"""The persistent cooperative PCG (one launch per solve, group barriers) is
bit-identical to the launch-per-phase loop, for solves through the drop-in
API (generic CSR, identity/Jacobi, history) and the level-batched solver."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

_SCRIPT = r"""
import sys, numpy as np, scipy.sparse as sp
sys.path.insert(0, sys.argv[1])
import paper_1705_02003_b200 as uq
out = []
cfg = uq.CONFIGS["C1"]
s = cfg.make_solver()
ys = np.random.default_rng(3).uniform(-1, 1, (5, cfg.ensemble_size, cfg.n_modes))
r = s.solve_groups(ys)
out += [r.iterations.ravel().astype(float), r.qoi.ravel()]
rng = np.random.default_rng(7)
n = 60
mask = np.triu(rng.random((n, n)) < 0.1, 1)
base = np.where(mask, rng.uniform(-1, 1, (n, n)), 0.0); base = base + base.T
lanes = []
for _ in range(3):
    v = base * rng.uniform(0.2, 1.0)
    np.fill_diagonal(v, np.abs(v).sum(axis=1) + 1.0)
    lanes.append(sp.csr_matrix(v))
ens = uq.EnsembleCsrMatrix.from_scipy_lanes(lanes)
res = uq.ensemble_pcg(ens, rng.standard_normal((3, n)), tol=1e-11, maxit=500, record_history=True)
out += [res.solution.ravel(), res.iterations_per_lane.astype(float),
        np.concatenate(res.residual_history)]
np.save(sys.argv[2], np.concatenate(out))
"""


def test_persistent_bitwise_equals_launch_loop(tmp_path):
    got = {}
    # cluster barriers, cooperative barriers, host-polled launch loop, graph launch loop
    for mode in ("2", "1", "0", "0g"):
        env = dict(os.environ, UQG_PCG_PERSISTENT=mode[0], UQG_PCG_GRAPH=str(int(mode == "0g")))
        dst = tmp_path / f"p{mode}.npy"
        subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT), str(dst)], env=env, check=True,
                       timeout=600)
        got[mode] = np.load(dst)
    assert got["1"].shape == got["0"].shape
    assert np.array_equal(got["1"], got["0"])
    assert np.array_equal(got["2"], got["0"])
    assert np.array_equal(got["0g"], got["0"])


@pytest.mark.parametrize("graph", ["0", "1"])
def test_reference_semantics_through_the_launch_loop(graph):
    """The PCG semantics tests (reference goldens, trivial systems, frozen and
    breakdown lanes, acceptance criterion 1) re-run with the small systems
    forced through the launch loop - deferred solution update included, host-
    polled or as one graph launch - instead of the persistent kernel they take
    by default."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, UQG_PCG_PERSISTENT="0", UQG_X_DEFER="4", UQG_PCG_GRAPH=graph)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        str(root / "tests" / "test_gpu_parity.py"), "-k",
                        "pcg_matches_reference_golden or trivial_systems or subnormal or "
                        "nonfinite or acceptance_crit1 or duplicated_lanes or companions"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
