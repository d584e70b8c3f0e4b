"""Row-partitioned operator: R partitions whose gathers read the
owner partition's block.  On one device every partitioned code path is checked
against the unpartitioned run and the reference goldens: T_m blocks bit-exact,
moments within the usual tolerances, for several R, with and without the hub
path."""

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from conftest import GRAPH_CASES
from paper_1905_09758_b200 import _lib
from paper_1905_09758_b200.partition import PartitionedOperator, balanced_bounds

pytestmark = pytest.mark.gpu


def _graph(golden, name):
    n = int(golden[f"{name}/n"])
    rp, ci = golden[f"{name}/row_ptr"], golden[f"{name}/col_idx"]
    return kp.GraphCSR(n=n, row_ptr=rp, col_idx=ci, weights=np.ones(ci.size),
                       is_weighted=False)


def _normwise(got, want):
    return np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300)


def test_balanced_bounds():
    rp = np.array([0, 5, 5, 6, 20, 21, 22], dtype=np.int64)
    b = balanced_bounds(rp, 3)
    assert b[0] == 0 and b[-1] == 6 and np.all(np.diff(b) >= 0)


@pytest.mark.parametrize("name", ["er200", "ba300", "ba_p64", "grid4x5"])
@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
@pytest.mark.parametrize("heavy", [None, "3"])
def test_partitioned_blocks_and_moments(golden, kpm_ctx, monkeypatch, name, nparts, heavy):
    if heavy:
        monkeypatch.setenv("KPM_HEAVY_DEGREE", heavy)
    g = _graph(golden, name)
    z = golden[f"{name}/probes"]
    nz, seed, m_dos, m_pdos = golden[f"{name}/meta"].tolist()
    pop = PartitionedOperator.from_graph(g, nparts)
    rp, ci, dinv = pop.export()
    assert np.array_equal(rp, g.row_ptr) and np.array_equal(ci.astype(np.int64), g.col_idx)
    probes = kp.ProbeMatrix(g.n, nz, "rademacher", seed, columns=z)
    for s in sorted(int(k.split("/T")[1]) for k in golden if k.startswith(f"{name}/T")):
        t = pop.step_blocks(probes, _lib.MODE_DOS_DIRECT, s, 2 * s + 2)
        assert np.array_equal(t, golden[f"{name}/T{s}"]), (name, nparts, s)
    c = pop.dos_contrib(probes, m_dos, doubling=False)
    assert _normwise(c, golden[f"{name}/dos_contrib"]) <= 1e-12
    for doubling in (True, False):
        mom = pop.dos_moments(probes, m_dos, doubling=doubling)
        assert _normwise(mom.values, golden[f"{name}/dos_values"]) <= 1e-9
    pd = pop.pdos_moments(probes, m_pdos)
    assert np.max(np.abs(pd.values - golden[f"{name}/pdos_values"])) <= 1e-12


def test_partitioned_rmat_matches_unpartitioned(kpm_ctx):
    full = kp.DeviceGraph.rmat(14, 16, 2)
    pop = PartitionedOperator.rmat(14, 16, 2, nparts=4)
    rp, ci, dinv = pop.export()
    frp, fci, fdinv = full.export()
    assert np.array_equal(rp, frp) and np.array_equal(ci, fci) and np.array_equal(dinv, fdinv)
    probes = kp.make_probes(full.n, 96, "rademacher", seed=2)  # device-generated rows
    sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(full), (-1.0, 1.0))
    want = kp.dos_contrib(sop, probes, 30, doubling=False)
    got = pop.dos_contrib(probes, 30, doubling=False)
    assert _normwise(got, want) <= 1e-12
    m_full = kp.dos_moments(sop, probes, 60)
    m_part = pop.dos_moments(probes, 60)
    assert _normwise(m_part.values, m_full.values) <= 1e-9
    assert np.array_equal(pop.step_blocks(probes, _lib.MODE_DOS_DOUBLING, 3, 8),
                          PartitionedOperator([full], [0, full.n]).step_blocks(
                              probes, _lib.MODE_DOS_DOUBLING, 3, 8))
