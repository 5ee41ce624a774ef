"""bench.py's CPU legs run without a GPU: the reference arm (the oracle port on
all host cores) prints one well-formed JSON line; the byte model matches
SURVEY.md 8d."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_runs_on_cpu():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config",
                        "C1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["metric"].startswith("ensemble sample-solves/s")
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")  # reference: baseline/_ref staged


def test_byte_model_matches_survey():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1705_02003_b200.configs import get
    bm = bench.bytes_model(get("C2"))
    assert bm["spmv"] == 59688364  # B_spmv at C2 = 59.7 MB
    assert abs(bm["pcg_iter"] - 151.2e6) < 0.1e6  # 151.2 MB
    assert bm["spmv"] + bm["update"] + bm["dir"] == bm["pcg_iter_moved"] < bm["pcg_iter"]
    assert bm["operator"] == "csr"


def test_byte_model_faces():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1705_02003_b200.configs import get

    class Op:  # the face-form FV2D operator's byte-relevant attributes
        faces, n_op = True, 256 * 255
    cfg = get("C2")
    bm = bench.bytes_model(cfg, Op())
    S, N = cfg.ensemble_size, cfg.n_dofs
    assert bm["operator"] == "fv2d faces"
    assert bm["spmv"] == 8 * S * (256 * 255) + 16 * S * N
    assert bm["pcg_iter"] == 8 * S * (256 * 255 + 13 * N)


def test_byte_model_deferred_update():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1705_02003_b200.configs import get

    cfg = get("C2")
    S, N = cfg.ensemble_size, cfg.n_dofs
    one = bench.bytes_model(cfg, kx=1)
    four = bench.bytes_model(cfg, kx=4)
    assert one["dir"] == 48 * S * N and "flush" not in one
    assert four["dir"] == int(5.5 * 8 * S * N) and four["flush"] == 4
    assert four["pcg_iter_moved"] < one["pcg_iter_moved"]
