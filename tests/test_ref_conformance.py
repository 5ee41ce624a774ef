"""The reference's own hot-path test modules, run UNMODIFIED against the
drop-ins.

``tools/stage_reference.py`` (called by ``__graft_entry__.build()`` where
/root/reference exists) installs the reference into ``baseline/_ref`` and
copies its tests there; the ``uqgroup_dropin`` pytest plugin
(``tests/ref_conformance``) rebinds ``uqgroup``'s hot-path names to
``paper_1705_02003_b200`` before collection.  Targets:
``pkg/tests/test_ensemble.py:41-248`` (container, SpMV bitwise vs scipy,
Jacobi, special cases, counts vs the scalar solver, lane independence,
freeze / breakdown, histories, hypothesis property) and
``pkg/tests/test_grouping.py:37-292`` (plans, ties, padding, validation, and
the reference's R accounting fed with the drop-in's plans) and
``pkg/tests/test_fem3d.py:43-185`` (the reference's 3D operator assembled on
the device: Kronecker oracle, stencil, symmetry, SPD, bitwise duplicate
lanes, direct-solve QoI, Laplacian centre value).
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
TESTS = REF / "ref_tests"
MODULES = ["test_ensemble.py", "test_grouping.py", "test_fem3d.py"]

staged = pytest.mark.skipif(not (REF / "uqgroup").exists() or not TESTS.exists(),
                            reason="reference not staged (tools/stage_reference.py)")


def _run(args, tmp_path, timeout=1200):
    (tmp_path / "pytest.ini").write_text("[pytest]\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [str(REF), str(TESTS), str(ROOT / "tests" / "ref_conformance"), str(ROOT)]),
        PYTHONDONTWRITEBYTECODE="1")
    return subprocess.run([sys.executable, "-m", "pytest", "-c", str(tmp_path / "pytest.ini"),
                           "--rootdir", str(tmp_path), "-p", "no:cacheprovider",
                           "-p", "uqgroup_dropin", *args], env=env, cwd=tmp_path,
                          capture_output=True, text=True, timeout=timeout)


@staged
def test_plugin_binds_the_dropins(tmp_path):
    """CPU: the plugin imports and rebinds (no compute)."""
    probe = tmp_path / "test_probe.py"
    probe.write_text(
        "import uqgroup, paper_1705_02003_b200 as uq\n"
        "def test_bound():\n"
        "    assert uqgroup.ensemble_pcg is uq.ensemble_pcg\n"
        "    assert uqgroup.group_by_key is uq.group_by_key\n"
        "    assert uqgroup.EnsembleCsrMatrix is uq.EnsembleCsrMatrix\n"
        "    assert isinstance(uq.EnsembleError('x'), uqgroup.EnsembleError)\n"
        "    assert isinstance(uq.GroupingError('x'), uqgroup.GroupingError)\n"
        "    assert isinstance(uq.FemError('x'), uqgroup.FemError)\n")
    r = _run(["-q", str(probe)], tmp_path)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@staged
@pytest.mark.gpu
@pytest.mark.parametrize("module", MODULES)
def test_reference_module_passes_against_dropins(module, tmp_path):
    r = _run(["-q", str(TESTS / module)], tmp_path)
    tail = r.stdout[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) > 0, tail
    print(f"{module}: {m.group(0)}")
