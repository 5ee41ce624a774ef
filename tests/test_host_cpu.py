"""Host-side logic that runs without a GPU: ABI surface, mesh/graph, field setup,
sparse-grid keys, plan validation, configs."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import field2d, fv2d as ofv
from paper_1705_02003_b200 import _lib, build_field, configs
from paper_1705_02003_b200.fv2d import StructuredMesh2D
from paper_1705_02003_b200.grouping import GroupingPlan
from paper_1705_02003_b200.errors import GroupingError
from paper_1705_02003_b200.sparse_grid import SparseGrid

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "uqg.h").read_text()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(uqg_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()  # loading needs no GPU
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table and header disagree"
    assert lib.uqg_version() == 1
    assert lib.uqg_pcg_workspace_bytes(100, 460, 8, 2) > 3 * 2 * 100 * 8 * 8


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_null_args_rejected_without_device():
    lib = _lib.load()
    rc = lib.uqg_spmv(None, 10, 10, 0, 2, 1, None, None, None, None, None, None)
    assert rc == _lib.UQG_EINVAL and "NULL" in _lib.last_error()


@pytest.mark.parametrize("n", [2, 3, 8, 64])
def test_mesh_graph_matches_oracle(n):
    m, o = StructuredMesh2D(n), ofv.Mesh2D(n)
    assert np.array_equal(m.row_offsets, o.row_offsets)
    assert np.array_equal(m.col_indices, o.col_indices)
    assert m.nnz == o.nnz == 5 * (n - 1) ** 2 - 4 * (n - 1)
    assert np.array_equal(m.node_coords(), o.node_points)


def test_config_sizes_match_survey():
    want = {"C1": (3969, 19593), "C2": (65025, 324105), "C3": (261121, 1303561),
            "C4": (1046529, 5228553), "C5": (4190209, 20942857)}
    for k, (N, nnz) in want.items():
        c = configs.get(k)
        assert (c.n_dofs, c.nnz) == (N, nnz)


@pytest.mark.parametrize("delta,sigma,M", [(0.2, 1.0, 3), (0.1, 1.5, 6), (0.05, 2.0, 10)])
def test_field_setup_bit_identical_to_oracle(delta, sigma, M):
    f = build_field(delta, sigma, M, 0.0)
    o = field2d.KL2D.select(delta, sigma, M, 0.0)
    assert f.modes == o.modes and np.array_equal(f.eigenvalues, o.eigenvalues)
    mesh = StructuredMesh2D(16)
    tab = f.mode_values(mesh.node_coords())
    assert np.array_equal(tab, o.mode_table(ofv.Mesh2D(16).node_points))
    t1 = f.node_tables(16)
    for k, (p, q) in enumerate(f.modes):  # separable rebuild == dense table, bitwise
        assert np.array_equal((t1[p][:, None] * t1[q][None, :]).ravel(), tab[k])


def test_sparse_grid_reproduces_reference_keys(c1_golden):
    """Fed the reference's per-sample results, the host grid yields the same
    level batches and bit-identical surrogate keys (grouping inputs)."""
    cfg = c1_golden["config"]
    g = SparseGrid(cfg["n_modes"])
    batch = g.add_initial_levels(cfg["initial_level"])
    for lv in c1_golden["levels"]:
        start = len(g) - len(batch)
        ids = list(range(start, len(g)))
        assert ids == lv["ids"]
        coords = g.node_coords()[start:]
        assert np.array_equal(coords, np.array(lv["coords"]))
        if lv["predicted"] is not None:
            assert np.array_equal(g.evaluate("iterations", coords, n_nodes=start),
                                  np.array(lv["predicted"]))
        g.fit("qoi", dict(zip(ids, lv["qoi"])))
        g.fit("iterations", dict(zip(ids, lv["iterations"])))
        batch, _ = g.refine(cfg["tau"], "qoi", cfg["n_max"])
        if not batch:
            break


def test_initial_grid_sizes():
    for M, L, n in ((3, 4, 297), (4, 5, 2441), (3, 0, 8), (10, 0, 1024)):
        g = SparseGrid(M)
        g.add_initial_levels(L)
        assert len(g) == n


def test_plan_validation():
    with pytest.raises(GroupingError):
        GroupingPlan(0, 2, ((1, 1), (2, 3)), (1, 0), "nat")
    with pytest.raises(GroupingError):
        GroupingPlan(0, 3, ((1, 2),), (0,), "nat")
    with pytest.raises(GroupingError):
        GroupingPlan(0, 3, ((1, 2, 9),), (1,), "nat")
    p = GroupingPlan(0, 4, ((7, 8, 9, 10), (11, 11, 11, 11)), (0, 3), "nat")
    assert p.n_samples == 5 and p.sample_ids() == [7, 8, 9, 10, 11]


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1705_02003_b200 import DeviceError, group_natural
    with pytest.raises(DeviceError):
        group_natural([1, 2, 3], 2)


def test_nkern_matches_header():
    """The profile arrays the bindings allocate are UQG_NKERN long: the library
    writes every entry (a shorter array corrupted the host heap)."""
    import re

    from paper_1705_02003_b200 import _lib

    h = (ROOT / "include" / "uqg.h").read_text()
    assert int(re.search(r"#define UQG_NKERN (\d+)", h).group(1)) == _lib.NKERN
