"""Per-node histograms on the device against fixtures
written by the reference (tests/golden/make_density_golden.py):
pdos_moments + histogram_from_moments on a BA and an ER graph."""

import os

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from oracle import netdos_oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "density.npz"))
TAGS = {"ba_rademacher": ("ba", "rademacher", 24, 60), "er_gaussian": ("er", "gaussian", 10, 33)}
EDGES = np.array([-1.0, -0.7, -0.1, 0.0, 0.25, 0.9, 1.0])
CALLS = {
    "h50": dict(bins=50, negativity_tol=1.0),
    "h50tol": dict(bins=50),
    "h7raw": dict(bins=7, damping=False),
    "hedges": dict(edges=EDGES, negativity_tol=1.0),
    "neg": dict(bins=80, damping=False, negativity_tol=1e-9),
    "rawh20": dict(bins=20, negativity_tol=10.0),
}


def _moments(tag, key):
    vals = GOLD[f"{tag}_raw_values" if key == "rawh20" else f"{tag}_values"]
    return kp.ChebMoments("per-node", vals, kp.ScaleMap(0.0, 1.0), {})


def _graph(name):
    rp, ci = GOLD[f"{name}_row_ptr"], GOLD[f"{name}_col_idx"]
    rows = np.repeat(np.arange(rp.shape[0] - 1), np.diff(rp))
    keep = rows < ci
    return kp.build_csr(list(zip(rows[keep].tolist(), ci[keep].tolist())), n=rp.shape[0] - 1)


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("tag", sorted(TAGS))
def test_oracle_per_node_masses_match_reference(tag):
    """The oracle's restated `coef @ table` reproduces the reference's
    per-node masses (pins the checker used by the GPU tests)."""
    edges, got = orc.histogram_masses(GOLD[f"{tag}_values"], bins=50)
    assert np.array_equal(edges, GOLD[f"{tag}_h50_edges"])
    assert np.array_equal(got, GOLD[f"{tag}_h50_masses"])


def test_fixture_contents():
    for tag in TAGS:
        assert f"{tag}_neg_error" in GOLD and f"{tag}_h50tol_error" in GOLD
        assert GOLD[f"{tag}_values"].shape[1] == TAGS[tag][3] + 1


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(CALLS))
@pytest.mark.parametrize("tag", sorted(TAGS))
def test_device_histogram_of_reference_moments(tag, key, kpm_ctx):
    """histogram_from_moments on per-node moments runs the device kernel;
    same masses (fp64, only the summation order differs), normalization
    bit-exact, same negativity errors."""
    mom = _moments(tag, key)
    err = GOLD.get(f"{tag}_{key}_error")
    if err is not None:
        with pytest.raises(ValueError) as ei:
            kp.histogram_from_moments(mom, **CALLS[key])
        assert str(ei.value) == str(err)
        return
    h = kp.histogram_from_moments(mom, **CALLS[key])
    ref = GOLD[f"{tag}_{key}_masses"]
    assert h.masses.shape == ref.shape
    assert np.abs(h.masses - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
    assert np.array_equal(h.normalization, GOLD[f"{tag}_{key}_norm"])
    assert np.array_equal(h.edges, GOLD[f"{tag}_{key}_edges"])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(TAGS))
def test_pdos_histogram_pipeline_matches_reference(tag, kpm_ctx):
    """LDOS recurrence + binning without the moments leaving HBM: per-row
    L1 distance to the reference's histograms <= 1e-6."""
    name, kind, nz, m = TAGS[tag]
    g = _graph(name)
    sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(g), (-1.0, 1.0))
    z = kp.make_probes(g.n, nz, kind, seed=5)
    h = kp.pdos_histogram(sop, z, m, bins=50, negativity_tol=1.0)
    ref = GOLD[f"{tag}_h50_masses"]
    assert np.abs(h.masses - ref).sum(axis=1).max() <= 1e-6
    assert np.abs(h.normalization - GOLD[f"{tag}_h50_norm"]).max() <= 1e-12
    with pytest.raises(ValueError, match="series is not a valid density"):
        kp.pdos_histogram(sop, z, m, bins=50)
    hr = kp.pdos_histogram(sop, z, m, bins=20, negativity_tol=10.0, normalized=False)
    assert np.abs(hr.masses - GOLD[f"{tag}_rawh20_masses"]).sum(axis=1).max() <= 1e-6
    # batched probes take the host-combined path, same histograms
    hb = kp.pdos_histogram(sop, z, m, bins=50, negativity_tol=1.0, batch=nz // 2)
    assert np.abs(hb.masses - h.masses).max() <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,m_max,bins", [(1, 0, 1), (63, 17, 65), (200_003, 100, 50),
                                          (5000, 500, 130)])
def test_per_node_masses_shapes(n, m_max, bins, kpm_ctx):
    """Tile edges (rows, bins, moments not multiples of 64/64/16), host and
    device operands, against numpy's product."""
    rng = np.random.default_rng(n)
    vals = rng.standard_normal((n, m_max + 1))
    edges = np.linspace(-1, 1, bins + 1)
    table = kp.cheb_bin_masses(m_max, edges)
    damp = kp.jackson_coefficients(m_max)
    masses, norm, mn = kp.density.per_node_masses(vals, m_max, table, damp)
    ref = (vals * damp) @ table
    assert np.abs(masses - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    assert np.array_equal(norm, vals[:, 0] * damp[0])
    assert mn == pytest.approx(ref.min(), rel=1e-12, abs=1e-14)
    masses2, norm2, _ = kp.density.per_node_masses(vals, m_max, table, None)
    assert np.abs(masses2 - vals @ table).max() <= 1e-12 * max(1.0, np.abs(vals @ table).max())
    assert np.array_equal(norm2, vals[:, 0])


@pytest.mark.gpu
def test_per_node_masses_nan_propagates(kpm_ctx):
    vals = np.ones((100, 5))
    vals[37, 2] = np.nan
    table = kp.cheb_bin_masses(4, np.linspace(-1, 1, 4))
    masses, _, mn = kp.density.per_node_masses(vals, 4, table)
    assert np.isnan(mn) and np.isnan(masses[37]).all() and not np.isnan(masses[36]).any()
