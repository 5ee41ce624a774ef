"""Grouping keys on the device: the iteration surrogate
evaluated on the GPU equals the host (reference-order BLAS) keys bit for bit on
every level of the reference's studies; the anisotropy indicator matches the
reference formula; a study with device keys reproduces the golden plans."""

import json

import numpy as np
import pytest

import paper_1705_02003_b200 as uq
from conftest import GOLDEN
from paper_1705_02003_b200.field import anisotropy_indicator, anisotropy_indicators
from paper_1705_02003_b200.sparse_grid import SparseGrid

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("study,dim,init,tau,nmax", [
    ("c1_adaptive", 3, 0, 1e-5, 10_000),
    ("pde_test1_study", 4, 1, 1e-3, 600),
    ("pde_test2_study", 4, 1, 1e-3, 600),
])
def test_device_keys_bit_identical_to_host(study, dim, init, tau, nmax):
    doc = json.loads((GOLDEN / f"{study}.json").read_text())
    g = SparseGrid(dim)
    batch = g.add_initial_levels(init)
    checked = 0
    for lv in doc["levels"]:
        start = len(g) - len(batch)
        ids = list(range(start, len(g)))
        coords = g.node_coords()[start:]
        if lv["predicted"] is not None:
            host = g.evaluate("iterations", coords, n_nodes=start)
            dev = g.evaluate_device("iterations", coords, n_nodes=start)
            assert np.array_equal(host, dev)
            assert np.array_equal(dev, np.array(lv["predicted"]))
            # QoI channel: not exact arithmetic, agrees to rounding
            hq = g.evaluate("qoi", coords, n_nodes=start)
            dq = g.evaluate_device("qoi", coords, n_nodes=start)
            np.testing.assert_allclose(dq, hq, rtol=1e-12, atol=1e-12 * np.abs(hq).max())
            checked += 1
        g.fit("qoi", dict(zip(ids, lv["qoi"])))
        g.fit("iterations", dict(zip(ids, lv["iterations"])))
        batch, _ = g.refine(tau, "qoi", nmax)
        if not batch:
            break
    assert checked >= 2


def test_anisotropy_indicator_matches_reference_formula():
    f = uq.build_field(0.25, np.sqrt(300.0), 4, 0.1, sigma0_convention="kernel", dim=3)
    mesh = uq.StructuredMesh3D(8)
    probes = mesh.quad_points
    mv = f.mode_values(probes)
    ys = np.random.default_rng(4).uniform(-1, 1, (7, 4))
    got = anisotropy_indicators(f, ys, probes, mv)
    for s in range(7):
        a = f.a_min + f.a_hat(ys[s])[0] * np.exp((ys[s] * np.sqrt(f.eigenvalues)) @ mv)
        want = np.max(np.maximum(a, max(f.a_y, f.a_z)) / np.minimum(a, min(f.a_y, f.a_z)))
        assert abs(got[s] - want) <= 1e-13 * want
    assert anisotropy_indicator(f, ys[2], probes, mv) == got[2]


def test_study_with_device_keys_reproduces_golden(c1_golden):
    from paper_1705_02003_b200.driver import adaptive_run
    records, _, _ = adaptive_run(uq.CONFIGS["C1"], device_keys=True)
    for rec, gold in zip(records, c1_golden["levels"]):
        assert [list(g) for g in rec.ensembles] == gold["ensembles"]
        if gold["predicted"] is not None:
            assert np.array_equal(rec.predicted, np.array(gold["predicted"]))


@pytest.mark.parametrize("study,dim,init,tau,nmax", [
    ("c1_adaptive", 3, 0, 1e-5, 10_000),
    ("pde_test1_study", 4, 1, 1e-3, 600),
    ("pde_test2_study", 4, 1, 1e-3, 600),
])
def test_device_surplus_fit(study, dim, init, tau, nmax):
    """Surplus fitting on the device along the reference's
    studies: iteration-channel surpluses bit-identical to the host fit, QoI
    channel to rounding."""
    import copy

    doc = json.loads((GOLDEN / f"{study}.json").read_text())
    host = SparseGrid(dim)
    batch = host.add_initial_levels(init)
    for lv in doc["levels"]:
        start = len(host) - len(batch)
        ids = list(range(start, len(host)))
        dev = copy.deepcopy(host)
        host.fit("qoi", dict(zip(ids, lv["qoi"])))
        host.fit("iterations", dict(zip(ids, lv["iterations"])))
        dev.fit_device("qoi", dict(zip(ids, lv["qoi"])))
        dev.fit_device("iterations", dict(zip(ids, lv["iterations"])))
        assert np.array_equal(dev.surplus["iterations"], host.surplus["iterations"])
        hq = host.surplus["qoi"]
        np.testing.assert_allclose(dev.surplus["qoi"], hq, rtol=1e-11,
                                   atol=1e-12 * np.abs(hq).max())
        batch, _ = host.refine(tau, "qoi", nmax)
        if not batch:
            break


def test_study_with_device_keys_and_fit_matches_golden_plans(c1_golden):
    from paper_1705_02003_b200.driver import adaptive_run
    records, _, _ = adaptive_run(uq.CONFIGS["C1"], device_keys=True)
    assert len(records) == len(c1_golden["levels"])
    for rec, gold in zip(records, c1_golden["levels"]):
        assert [list(g) for g in rec.ensembles] == gold["ensembles"]
