"""Stage the reference for the conformance tests and the reference arm.

    python tools/stage_reference.py

Where /root/reference exists (the build container): installs the unmodified
reference package into ``baseline/_ref`` (the one offline install the task
allows: pip --no-index from /opt/wheelhouse, from a /tmp copy because the
build writes into its source tree) and copies its test modules to
``baseline/_ref/ref_tests``.  ``baseline/_ref`` is git-ignored but travels
to the GPU box with gpurun, where ``tests/test_ref_conformance.py`` runs
those modules against the drop-ins.  No-op elsewhere.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg")
DST = ROOT / "baseline" / "_ref"


def stage(force: bool = False) -> bool:
    if not REF.exists():
        return (DST / "uqgroup").exists()
    if force or not (DST / "uqgroup").exists():
        with tempfile.TemporaryDirectory() as tmp:
            src = Path(tmp) / "pkg"
            shutil.copytree(REF, src)
            subprocess.run([sys.executable, "-m", "pip", "install", "--no-index",
                            "--no-build-isolation", "--no-deps", "--find-links",
                            "/opt/wheelhouse", "--target", str(DST), "--upgrade", str(src)],
                           check=True, capture_output=True)
    tests = DST / "ref_tests"
    tests.mkdir(parents=True, exist_ok=True)
    for f in (REF / "tests").glob("*.py"):
        shutil.copy(f, tests / f.name)
    return True


if __name__ == "__main__":
    print("staged" if stage("--force" in sys.argv) else "reference not available")
