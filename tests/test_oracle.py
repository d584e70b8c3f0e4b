"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden).

The golden fixtures were written by the unmodified reference package (netdos
0.1.0 with its compiled Cython kernel) via tests/golden/make_golden.py.  These
CPU tests establish that the oracle -- the checker the GPU parity tests use --
reproduces the reference bit-for-bit where the reference is deterministic
(CSR, d^-1/2, operator values, T_m blocks, per-probe contributions, moments,
histograms, probes) and to 1e-13 where numpy's SIMD reduction order differs
(per-node sums).
"""

import hashlib

import numpy as np
import pytest

from conftest import GRAPH_CASES


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", GRAPH_CASES)
def test_csr_dinv_values_bitexact(golden, oracle, name):
    rp, ci = golden[f"{name}/row_ptr"], golden[f"{name}/col_idx"]
    n = int(golden[f"{name}/n"])
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = rows <= ci
    r2, c2 = oracle.csr_from_edges(n, rows[keep], ci[keep])
    assert np.array_equal(r2, rp) and np.array_equal(c2, ci)
    r3, c3 = oracle.csr_from_canonical(n, rows[keep], ci[keep])
    assert np.array_equal(r3, rp) and np.array_equal(c3, ci)
    assert np.array_equal(oracle.degrees(rp), golden[f"{name}/degrees"])
    data = oracle.normadj_values(rp, ci)
    assert np.array_equal(data, golden[f"{name}/op_data"])
    assert np.array_equal(golden[f"{name}/op_indptr"], rp)


def test_canonical_dedup_csr(golden, oracle):
    u, v = golden["canon/u"], golden["canon/v"]
    r, c = oracle.csr_from_edges(700, u, v)
    assert np.array_equal(r, golden["canon/row_ptr"])
    assert np.array_equal(c, golden["canon/col_idx"])
    a, b = oracle.canonical_pairs(u, v)
    r2, c2 = oracle.csr_from_canonical(700, a, b)
    assert np.array_equal(r2, golden["canon/row_ptr"]) and np.array_equal(c2, c)


@pytest.mark.parametrize("name", GRAPH_CASES)
@pytest.mark.parametrize("engine", ["c", "ref"])
def test_recurrence_blocks_bitexact(golden, oracle, name, engine):
    if engine == "ref" and oracle.ref_spmv() is None:
        pytest.skip("oracle/_ref not built")
    rp, ci, data = (golden[f"{name}/row_ptr"], golden[f"{name}/col_idx"],
                    golden[f"{name}/op_data"])
    z = golden[f"{name}/probes"]
    op = oracle.CSROp(rp, ci, data, engine=engine)
    for key in [k for k in golden if k.startswith(f"{name}/T")]:
        steps = int(key.split("/T")[1])
        assert np.array_equal(oracle.recurrence_block(op, z, steps), golden[key]), key
        assert np.array_equal(oracle.c_recurrence_block(rp, ci, data, z, steps), golden[key])


@pytest.mark.parametrize("name", GRAPH_CASES)
def test_dos_contrib_and_moments_bitexact(golden, oracle, name):
    rp, ci, data = (golden[f"{name}/row_ptr"], golden[f"{name}/col_idx"],
                    golden[f"{name}/op_data"])
    z = golden[f"{name}/probes"]
    nz, seed, m_dos, m_pdos = golden[f"{name}/meta"].tolist()
    want = golden[f"{name}/dos_contrib"]
    got = oracle.c_dos_contrib(rp, ci, data, z, m_dos)
    assert np.array_equal(got, want)
    got_np = oracle.dos_contrib(oracle.CSROp(rp, ci, data), z, m_dos)
    assert np.array_equal(got_np, want)
    vals = oracle.dos_values(got, 1.0 / nz, float(rp.shape[0] - 1))
    assert np.array_equal(vals, golden[f"{name}/dos_values"])


@pytest.mark.parametrize("name", GRAPH_CASES)
def test_ldos_values(golden, oracle, name):
    rp, ci, data = (golden[f"{name}/row_ptr"], golden[f"{name}/col_idx"],
                    golden[f"{name}/op_data"])
    z = golden[f"{name}/probes"]
    nz, seed, m_dos, m_pdos = golden[f"{name}/meta"].tolist()
    want = golden[f"{name}/pdos_values"]
    num = oracle.c_ldos_num(rp, ci, data, z, m_pdos)
    got = oracle.pdos_values(num, z)
    assert np.max(np.abs(got - want)) <= 1e-13
    num2 = oracle.ldos_num(oracle.CSROp(rp, ci, data), z, m_pdos)
    assert np.array_equal(oracle.pdos_values(num2, z), want)


@pytest.mark.parametrize("name", GRAPH_CASES)
def test_histogram_bitexact(golden, oracle, name):
    edges, masses = oracle.histogram_masses(golden[f"{name}/dos_values"], bins=50)
    assert np.array_equal(edges, golden[f"{name}/hist_edges"])
    assert np.array_equal(masses, golden[f"{name}/hist_masses"])


def test_explicit_values_mode(golden, oracle):
    rp, ci, data = golden["lap60/indptr"], golden["lap60/indices"], golden["lap60/data"]
    shift, scale = golden["lap60/shift_scale"].tolist()
    z = golden["lap60/probes"]
    op = oracle.CSROp(rp, ci, data, shift, scale)
    assert np.array_equal(oracle.recurrence_block(op, z, 3), golden["lap60/T3"])
    assert np.array_equal(oracle.c_recurrence_block(rp, ci, data, z, 3, shift, scale),
                          golden["lap60/T3"])
    contrib = oracle.c_dos_contrib(rp, ci, data, z, 30, shift, scale)
    vals = oracle.dos_values(contrib, 1.0 / z.shape[1], float(z.shape[0]))
    assert np.array_equal(vals, golden["lap60/dos_values"])


@pytest.mark.parametrize("kind", ["rademacher", "gaussian", "hadamard"])
def test_probe_generators_bitexact(golden, oracle, kind):
    assert np.array_equal(oracle.make_probes(1000, 8, kind, seed=17), golden[f"probes/{kind}"])


def test_standard_basis_and_column_stability(golden, oracle):
    assert np.array_equal(oracle.make_probes(6, 4, "standard-basis"), golden["probes/std_basis"])
    full = golden["probes/rademacher"]
    for j in range(8):
        assert np.array_equal(oracle.rademacher_column(1000, 17, j), full[:, j])


def test_motif_projection(golden, golden_meta, oracle):
    # the filtered block is the projection of the probes onto the complement
    # of the detected eigenvectors: its Gram with itself equals P^T(I-UU^T)P
    z, f = golden["motif/probes"], golden["motif/filtered"]
    assert z.shape == f.shape
    removed = sum(golden_meta["motif"]["removed"].values())
    assert removed == 75
    # deflation only moves mass inside supports of removed vectors
    changed = np.flatnonzero(np.any(z != f, axis=1))
    assert changed.size > 0


def test_c1_oracle_digests(golden_meta, oracle):
    from paper_1905_09758_b200.testkit import erdos_renyi
    g = erdos_renyi(10000, 1e-3, seed=0)
    c1 = golden_meta["c1"]
    assert _sha(g.row_ptr) == c1["row_ptr"] and _sha(g.col_idx) == c1["col_idx"]
    data = oracle.normadj_values(g.row_ptr, g.col_idx)
    assert _sha(data) == c1["dinv_data"]
    z = oracle.make_probes(10000, 20, "rademacher", seed=0)
    assert _sha(z) == c1["probes"]
    for s in (1, 2, 7):
        assert _sha(oracle.c_recurrence_block(g.row_ptr, g.col_idx, data, z, s)) == c1[f"T{s}"]


def test_c1_oracle_moments(golden, oracle):
    from paper_1905_09758_b200.testkit import erdos_renyi
    g = erdos_renyi(10000, 1e-3, seed=0)
    data = oracle.normadj_values(g.row_ptr, g.col_idx)
    z = oracle.make_probes(10000, 20, "rademacher", seed=0)
    contrib = oracle.c_dos_contrib(g.row_ptr, g.col_idx, data, z, 200, threads=4)
    vals = oracle.dos_values(contrib, 1.0 / 20, 10000.0)
    assert np.array_equal(vals, golden["c1/dos_values"])
    _, masses = oracle.histogram_masses(vals, bins=100)
    assert np.array_equal(masses, golden["c1/hist_masses"])


def test_rmat_generator_deterministic(oracle):
    u1, v1 = oracle.rmat_edges(10, 16 << 10, seed=2, threads=1)
    u2, v2 = oracle.rmat_edges(10, 16 << 10, seed=2, threads=4)
    assert np.array_equal(u1, u2) and np.array_equal(v1, v2)
    assert u1.min() >= 0 and u1.max() < 1024 and v1.max() < 1024
    # quadrant a (top-left) dominates: first-level bits are 0 ~57% of draws
    top = ((u1 >> 9) == 0) & ((v1 >> 9) == 0)
    assert 0.53 < top.mean() < 0.61
    # a prefix/slice of the stream is reproducible on its own
    u3, v3 = oracle.rmat_edges(10, 16 << 10, seed=2, e0=100, count=50, threads=1)
    assert np.array_equal(u3, u1[100:150]) and np.array_equal(v3, v1[100:150])
