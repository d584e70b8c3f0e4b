"""Device Lanczos / Gauss quadrature against fixtures
written by the reference (tests/golden/make_lanczos_golden.py), plus ports of
the reference's tests/test_lanczos.py.

Tolerances: the SpMV is bit-identical to the reference's apply; the dot
products / Gram-Schmidt sums run in a different (fixed) order than numpy's
BLAS, so alphas, betas, Ritz nodes and weights agree to 1e-9 relative
(observed ~1e-13); GQL histograms to L1 1e-9."""

import os

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from oracle import netdos_oracle as orc
from paper_1905_09758_b200 import testkit

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "lanczos.npz"))
KINDS = ("adjacency", "laplacian", "normalized-adjacency", "normalized-laplacian")
GRAPHS = ("er", "ba")
gpu = pytest.mark.gpu


def _graph(name):
    rp, ci = GOLD[f"{name}/row_ptr"], GOLD[f"{name}/col_idx"]
    rows = np.repeat(np.arange(rp.shape[0] - 1), np.diff(rp))
    keep = rows < ci
    return kp.build_csr(list(zip(rows[keep].tolist(), ci[keep].tolist())), n=rp.shape[0] - 1)


def close(a, b, tol=1e-9):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    assert np.abs(a - b).max(initial=0.0) <= tol * max(1.0, np.abs(b).max(initial=0.0))


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gname", GRAPHS)
def test_oracle_lanczos_matches_reference(gname, kind):
    """The oracle's restated lanczos_factorize (numpy, the reference's own
    arithmetic over the C oracle's SpMV) reproduces the reference bit for bit."""
    g = _graph(gname)
    op = kp.build_operator(g, kind)
    ip, ix, dd = op.csr_arrays()
    a, b, exh, _ = orc.lanczos_factorize(lambda x: orc.csr_matvec(ip, ix, dd, x), GOLD[f"{gname}/z"], 40)
    assert np.array_equal(a, GOLD[f"{gname}/{kind}/alphas"])
    assert np.array_equal(b, GOLD[f"{gname}/{kind}/betas"])
    assert exh == bool(GOLD[f"{gname}/{kind}/exhausted"])
    nodes, weights = orc.ritz_rule(*orc.lanczos_factorize(
        lambda x: orc.csr_matvec(ip, ix, dd, x), GOLD[f"{gname}/z"], 12)[:2])
    assert np.array_equal(nodes, GOLD[f"{gname}/{kind}/q_nodes"])
    assert np.array_equal(weights, GOLD[f"{gname}/{kind}/q_weights"])


def test_quadrature_to_moments_host():
    q = kp.RitzQuadrature(nodes=np.array([0.0]), weights=np.array([1.0]), z_norm_sq=1.0)
    assert np.allclose(kp.quadrature_to_cheb_moments(q, 5).values, [1, 0, -1, 0, 1, 0],
                       atol=1e-15)
    q2 = kp.RitzQuadrature(nodes=np.array([-1.0, 1.0]), weights=np.array([0.5, 0.5]),
                           z_norm_sq=1.0)
    assert np.allclose(kp.quadrature_to_cheb_moments(q2, 5).values, [1, 0, 1, 0, 1, 0],
                       atol=1e-15)
    with pytest.raises(ValueError, match="outside"):
        kp.quadrature_to_cheb_moments(
            kp.RitzQuadrature(nodes=np.array([1.5]), weights=np.array([1.0]), z_norm_sq=1.0), 3)


# ------------------------------------------------------------------ GPU
@gpu
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gname", GRAPHS)
def test_device_lanczos_matches_reference(gname, kind, kpm_ctx):
    g = _graph(gname)
    op = kp.build_operator(g, kind)
    tag = f"{gname}/{kind}"
    z = GOLD[f"{gname}/z"]
    f = kp.lanczos_factorize(op, z, 40)
    assert f.exhausted == bool(GOLD[f"{tag}/exhausted"])
    close(f.alphas, GOLD[f"{tag}/alphas"])
    close(f.betas, GOLD[f"{tag}/betas"])
    close(kp.estimate_spectral_range(op, probe_seed=2, steps=60), GOLD[f"{tag}/range"])
    q = kp.lanczos_quadrature(op, z, 12)
    close(q.nodes, GOLD[f"{tag}/q_nodes"])
    close(q.weights, GOLD[f"{tag}/q_weights"])
    probes = kp.make_probes(g.n, 8, "rademacher", seed=3)
    h = kp.gql_dos(op, probes, 30, bins=40)
    close(h.edges, GOLD[f"{tag}/gql_edges"])
    assert np.abs(h.masses - GOLD[f"{tag}/gql_masses"]).sum() <= 1e-9
    assert h.normalization == pytest.approx(float(GOLD[f"{tag}/gql_norm"]), abs=1e-12)
    q = kp.gql_pdos(op, 7, 10)
    close(q.nodes, GOLD[f"{tag}/pdos_nodes"])
    close(q.weights, GOLD[f"{tag}/pdos_weights"])


@gpu
@pytest.mark.parametrize("gname", GRAPHS)
def test_device_gql_pipeline_and_scaled_operator(gname, kpm_ctx):
    g = _graph(gname)
    h = kp.gql_dos_pipeline(g, "laplacian", steps=25, nz=6, probe_kind="gaussian", seed=5,
                            bins=30)
    close(h.edges, GOLD[f"{gname}/pipeline_edges"])
    assert np.abs(h.masses - GOLD[f"{gname}/pipeline_masses"]).sum() <= 1e-9
    sop = kp.scaled_operator_for(g, "normalized-laplacian", seed=1)
    q = kp.lanczos_quadrature(sop, GOLD[f"{gname}/z"], 15)
    close(q.nodes, GOLD[f"{gname}/scaled_nodes"])
    close(q.weights, GOLD[f"{gname}/scaled_weights"])


@gpu
def test_exhausted_krylov_spaces(kpm_ctx):
    tri = kp.build_csr([(0, 1), (1, 2), (0, 2)])
    q = kp.lanczos_quadrature(kp.build_operator(tri, "adjacency"), np.ones(3), 5)
    assert q.exhausted and bool(GOLD["tri/exhausted"])
    close(q.nodes, GOLD["tri/nodes"], 1e-12)
    loop = kp.build_csr([(0, 1), (2, 2, 3.0)], allow_self_loops=True)
    q = kp.gql_pdos(kp.build_operator(loop, "adjacency"), 2, 4)
    assert q.exhausted and q.nodes.tolist() == [3.0] and q.weights.tolist() == [1.0]
    assert q.z_norm_sq == 1.0


@gpu
def test_block_columns_equal_single_runs(kpm_ctx):
    """k columns in one lockstep pass == k separate factorisations (each
    column's arithmetic is independent of the others, incl. breakdowns)."""
    g = kp.erdos_renyi(300, 0.03, seed=2)
    op = kp.build_operator(g, "laplacian")
    z = np.random.default_rng(1).standard_normal((g.n, 5))
    z[:, 3] = 0.0
    z[7, 3] = 1.0   # a basis vector: may exhaust early on its component
    facts = kp.lanczos.lanczos_factorize_block(op, z, 50)
    for c in range(5):
        f = kp.lanczos_factorize(op, z[:, c], 50)
        assert np.array_equal(f.alphas, facts[c].alphas)
        assert np.array_equal(f.betas, facts[c].betas)
        assert f.exhausted == facts[c].exhausted


@gpu
def test_larger_graph_vs_oracle(kpm_ctx):
    """R-MAT 14 Laplacian (16k nodes), 80 steps: device vs the oracle's
    restated factorisation; basis orthonormal."""
    dev = kp.DeviceGraph.rmat(14, 8, seed=3)
    g = dev.to_host()
    op = kp.build_operator(g, "laplacian")
    ip, ix, dd = op.csr_arrays()
    z = np.random.default_rng(4).standard_normal(g.n)
    a, b, exh, _ = orc.lanczos_factorize(lambda x: orc.csr_matvec(ip, ix, dd, x), z, 80)
    f = kp.lanczos_factorize(op, z, 80, keep_basis=True)
    assert f.exhausted == exh
    close(f.alphas, a, 1e-8)
    close(f.betas, b, 1e-8)
    gram = f.basis.T @ f.basis
    assert np.abs(gram - np.eye(f.steps)).max() <= 1e-8
    lo, hi = kp.estimate_spectral_range(op, steps=100)
    ev = np.linalg.eigvalsh(testkit.dense_matrix(op)) if g.n <= 4096 else None
    assert lo < 0.0 + 1e-6 and hi > 0.0
    if ev is not None:
        assert lo <= ev[0] + 1e-6 and hi >= ev[-1] - 1e-6


# ---------------------------------------- ports of reference tests/test_lanczos.py
@gpu
def test_single_step_is_rayleigh_quotient(kpm_ctx):
    path3 = kp.build_csr([(0, 1), (1, 2)])
    op = kp.build_operator(path3, "laplacian")
    z = np.random.default_rng(0).standard_normal(3)
    quad = kp.lanczos_quadrature(op, z, 1)
    h = testkit.dense_matrix(op)
    assert quad.nodes.shape == (1,)
    assert quad.nodes[0] == pytest.approx(z @ h @ z / (z @ z), abs=1e-12)
    assert quad.weights[0] == 1.0


@gpu
def test_gauss_exactness_random_pairs(kpm_ctx):
    rng = np.random.default_rng(7)
    for _ in range(20):
        n = int(rng.integers(8, 40))
        g = kp.erdos_renyi(n, 0.25, seed=int(rng.integers(1 << 30)))
        op = kp.build_operator(g, "adjacency")
        h = testkit.dense_matrix(op)
        z = rng.standard_normal(n)
        m = int(rng.integers(2, 7))
        quad = kp.lanczos_quadrature(op, z, m)
        assert quad.weights.sum() == pytest.approx(1.0, abs=1e-10)
        for k in range(2 * m):
            want = z @ np.linalg.matrix_power(h, k) @ z / (z @ z)
            assert quad.weights @ quad.nodes ** k == pytest.approx(want, rel=1e-9, abs=1e-9)


@gpu
def test_ritz_interlacing_in_step_count(kpm_ctx):
    g = kp.erdos_renyi(60, 0.1, seed=3)
    op = kp.build_operator(g, "normalized-adjacency")
    z = np.random.default_rng(2).standard_normal(60)
    prev = None
    for m in range(2, 12):
        nodes = np.sort(kp.lanczos_quadrature(op, z, m).nodes)
        if prev is not None:
            assert nodes[0] <= prev[0] + 1e-12 and nodes[-1] >= prev[-1] - 1e-12
        prev = nodes


@gpu
def test_gql_pdos_p3_center(kpm_ctx):
    path3 = kp.build_csr([(0, 1), (1, 2)])
    op = kp.build_operator(path3, "normalized-adjacency")
    quad = kp.gql_pdos(op, 1, steps=2)
    h = testkit.dense_matrix(op)
    for k in range(4):
        want = np.linalg.matrix_power(h, k)[1, 1]
        assert quad.weights @ quad.nodes ** k == pytest.approx(want, abs=1e-10)
    assert np.allclose(np.sort(quad.nodes), [-1.0, 1.0], atol=1e-10)


@gpu
def test_quadrature_moments_match_kpm_single_probe(kpm_ctx):
    g = kp.build_csr([(0, 1), (1, 2), (2, 3)])
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    probes = kp.make_probes(4, 1, "rademacher", seed=6)
    quad = kp.lanczos_quadrature(sop, probes.columns[:, 0], 4)
    mom_q = kp.quadrature_to_cheb_moments(quad, 7, scale_map=sop.scale_map)
    mom_k = kp.dos_moments(sop, probes, 7)
    assert np.abs(mom_q.values - mom_k.values).max() < 1e-8


@gpu
def test_zero_start_vector_rejected(kpm_ctx):
    op = kp.build_operator(kp.build_csr([(0, 1), (1, 2)]), "adjacency")
    with pytest.raises(ValueError, match="nonzero"):
        kp.lanczos_quadrature(op, np.zeros(3), 2)
    with pytest.raises(ValueError, match="steps"):
        kp.lanczos_factorize(op, np.ones(3), 0)


@gpu
def test_nan_operator_raises_spectral_range_error(kpm_ctx):
    op = kp.build_operator(kp.build_csr([(0, 1), (1, 2)]), "laplacian")
    bad = kp.operators.SymmetricCSROperator(op.n, op.indptr, op.indices,
                                            np.where(op.data > 1, np.nan, op.data), op.kind)
    with pytest.raises(kp.SpectralRangeError) as ei:
        kp.lanczos_factorize(bad, np.ones(3), 3)
    assert ei.value.iterations == 1
