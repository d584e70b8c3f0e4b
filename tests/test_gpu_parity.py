"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's golden fixtures.

Tolerances (north_star): CSR, degrees, d^-1/2 and every T_m block bit-exact;
global moments within normwise relative 1e-9 (direct estimator: 1e-12, it
differs from the reference only in the order of the final row sum);
per-node moments within 1e-12 absolute (|c| <= 1 + O(1/sqrt nz));
damped histograms within L1 1e-6.
"""

import ctypes

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from conftest import GRAPH_CASES
from paper_1905_09758_b200 import _lib
from paper_1905_09758_b200.kpm import Run

pytestmark = pytest.mark.gpu


def _graph(golden, name):
    n = int(golden[f"{name}/n"])
    rp, ci = golden[f"{name}/row_ptr"], golden[f"{name}/col_idx"]
    return kp.GraphCSR(n=n, row_ptr=rp, col_idx=ci, weights=np.ones(ci.size),
                       is_weighted=False)


def _normwise(got, want):
    return np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300)


def _d2h(ptr, shape, ctx):
    out = np.empty(shape)
    _lib.check(_lib.load().kpm_memcpy(ctx.handle, _lib.ptr(out), ptr, out.nbytes, 1))
    ctx.synchronize()
    return out


# ------------------------------------------------------------- graph loader
@pytest.mark.parametrize("name", GRAPH_CASES)
def test_device_loader_bitexact(golden, oracle, kpm_ctx, name):
    g = _graph(golden, name)
    u, v, _ = g.edge_list()
    # feed both orientations + duplicates: the loader canonicalises and dedups
    uu = np.concatenate([u, v, u])
    vv = np.concatenate([v, u, v])
    dev = kp.DeviceGraph.from_edges(g.n, uu, vv)
    rp, ci, dinv = dev.export()
    assert np.array_equal(rp, g.row_ptr)
    assert np.array_equal(ci.astype(np.int64), g.col_idx)
    assert np.array_equal(dinv, oracle.dinv_of(g.row_ptr))
    assert np.array_equal(np.diff(rp).astype(float), golden[f"{name}/degrees"])
    assert dev.max_degree == int(np.diff(g.row_ptr).max(initial=0))


def test_device_loader_canon_and_errors(golden, kpm_ctx):
    dev = kp.DeviceGraph.from_edges(700, golden["canon/u"], golden["canon/v"])
    rp, ci, _ = dev.export()
    assert np.array_equal(rp, golden["canon/row_ptr"])
    assert np.array_equal(ci.astype(np.int64), golden["canon/col_idx"])
    with pytest.raises(ValueError):
        kp.DeviceGraph.from_edges(5, [0, 1], [1, 7])
    empty = kp.DeviceGraph.from_edges(4, [], [])
    rp, ci, dinv = empty.export()
    assert rp.tolist() == [0] * 5 and ci.size == 0 and dinv.tolist() == [0.0] * 4
    loops = kp.DeviceGraph.from_edges(3, [0, 1, 2], [0, 2, 2], keep_loops=True)
    rp, ci, _ = loops.export()
    assert rp.tolist() == [0, 1, 2, 4] and ci.tolist() == [0, 2, 1, 2]


def test_rmat_device_matches_oracle(oracle, kpm_ctx):
    scale, ef, seed = 14, 16, 2
    m = ef << scale
    u, v = oracle.rmat_edges(scale, m, seed)
    rp, ci = oracle.csr_from_edges(1 << scale, u, v)
    dev = kp.DeviceGraph.rmat(scale, ef, seed)
    drp, dci, ddinv = dev.export()
    assert np.array_equal(drp, rp) and np.array_equal(dci.astype(np.int64), ci)
    assert np.array_equal(ddinv, oracle.dinv_of(rp))
    # raw draws too (device buffers through the C-ABI)
    ctx = kpm_ctx
    pu, pv = ctypes.c_void_p(), ctypes.c_void_p()
    L = _lib.load()
    cnt = 5000
    _lib.check(L.kpm_device_alloc(ctx.handle, 8 * cnt, ctypes.byref(pu)))
    _lib.check(L.kpm_device_alloc(ctx.handle, 8 * cnt, ctypes.byref(pv)))
    ta, tab, tabc = oracle.rmat_thresholds()
    _lib.check(L.kpm_rmat_edges(ctx.handle, scale, seed, ta, tab, tabc, 777, cnt, pu, pv))
    hu = np.empty(cnt, dtype=np.int64)
    hv = np.empty(cnt, dtype=np.int64)
    _lib.check(L.kpm_memcpy(ctx.handle, _lib.ptr(hu), pu, 8 * cnt, 1))
    _lib.check(L.kpm_memcpy(ctx.handle, _lib.ptr(hv), pv, 8 * cnt, 1))
    ctx.synchronize()
    L.kpm_device_free(ctx.handle, pu)
    L.kpm_device_free(ctx.handle, pv)
    assert np.array_equal(hu, u[777:777 + cnt]) and np.array_equal(hv, v[777:777 + cnt])


# ---------------------------------------------------------- recurrence core
@pytest.mark.parametrize("name", GRAPH_CASES)
@pytest.mark.parametrize("mode", [_lib.MODE_DOS_DIRECT, _lib.MODE_DOS_DOUBLING,
                                  _lib.MODE_LDOS])
def test_T_blocks_bitexact_vs_reference(golden, kpm_ctx, name, mode):
    g = _graph(golden, name)
    z = golden[f"{name}/probes"]
    dev = g.device()
    steps = sorted(int(k.split("/T")[1]) for k in golden if k.startswith(f"{name}/T"))
    run = Run(dev, z.shape[1], mode, 2 * max(steps) + 2)
    run.set_probe_block(z, z.shape[1])
    done = 0
    for s in steps:
        run.advance(s - done)
        done = s
        ptr, ld, kidx = run.block()
        assert kidx == s
        t = _d2h(ptr, (g.n, ld), kpm_ctx)[:, : z.shape[1]]
        assert np.array_equal(t, golden[f"{name}/T{s}"]), (name, s)
    run.free()


@pytest.mark.parametrize("name", GRAPH_CASES)
def test_dos_moments_vs_reference(golden, kpm_ctx, name):
    g = _graph(golden, name)
    z = golden[f"{name}/probes"]
    nz, seed, m_dos, m_pdos = golden[f"{name}/meta"].tolist()
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    probes = kp.with_columns(kp.make_probes(g.n, nz, "rademacher", seed), z)
    c_direct = kp.dos_contrib(sop, probes, m_dos, doubling=False)
    assert _normwise(c_direct, golden[f"{name}/dos_contrib"]) <= 1e-12
    for doubling in (False, True):
        mom = kp.dos_moments(sop, probes, m_dos, doubling=doubling)
        assert _normwise(mom.values, golden[f"{name}/dos_values"]) <= 1e-9
        h = kp.histogram_from_moments(mom, bins=50)
        assert np.abs(h.masses - golden[f"{name}/hist_masses"]).sum() <= 1e-6


@pytest.mark.parametrize("name", GRAPH_CASES)
def test_pdos_moments_vs_reference(golden, kpm_ctx, name):
    g = _graph(golden, name)
    z = golden[f"{name}/probes"]
    nz, seed, m_dos, m_pdos = golden[f"{name}/meta"].tolist()
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    probes = kp.with_columns(kp.make_probes(g.n, nz, "rademacher", seed), z)
    mom = kp.pdos_moments(sop, probes, m_pdos)
    assert mom.values.shape == (g.n, m_pdos + 1) and mom.values.flags.c_contiguous
    want = golden[f"{name}/pdos_values"]
    assert np.max(np.abs(mom.values - want)) <= 1e-12
    raw = kp.pdos_moments(sop, probes, m_pdos, normalized=False)
    assert np.max(np.abs(raw.values - want)) <= 1e-12  # +-1 probes: den = nz


def test_explicit_values_mode_vs_reference(golden, kpm_ctx):
    rp, ci, data = golden["lap60/indptr"], golden["lap60/indices"], golden["lap60/data"]
    shift, scale = golden["lap60/shift_scale"].tolist()
    z = golden["lap60/probes"]
    op = kp.SymmetricCSROperator(rp.shape[0] - 1, rp, ci, data, "laplacian")
    sop = kp.ScaledOperator(op, shift, scale, shift - scale, shift + scale)
    dev = sop.device_graph()
    run = Run(dev, z.shape[1], _lib.MODE_DOS_DIRECT, 5)
    run.set_probe_block(z, z.shape[1])
    run.advance(3)
    ptr, ld, _ = run.block()
    assert np.array_equal(_d2h(ptr, (z.shape[0], ld), kpm_ctx)[:, : z.shape[1]],
                          golden["lap60/T3"])
    run.free()
    probes = kp.ProbeMatrix(z.shape[0], z.shape[1], "gaussian", 8, columns=z)
    for doubling in (False, True):
        mom = kp.dos_moments(sop, probes, 30, doubling=doubling)
        assert _normwise(mom.values, golden["lap60/dos_values"]) <= 1e-9
    pd = kp.pdos_moments(sop, probes, 15)
    assert np.max(np.abs(pd.values - golden["lap60/pdos_values"])) <= 1e-10


# ------------------------------------------------------- native SpMM drop-in
@pytest.mark.parametrize("name", GRAPH_CASES + ["lap60"])
def test_csr_matvec_bitexact_vs_cython(golden, oracle, kpm_ctx, name):
    if name == "lap60":
        rp, ci, data = golden["lap60/indptr"], golden["lap60/indices"], golden["lap60/data"]
    else:
        rp, ci, data = (golden[f"{name}/op_indptr"], golden[f"{name}/op_indices"],
                        golden[f"{name}/op_data"])
    x = np.random.default_rng(1).standard_normal((rp.shape[0] - 1, 9))
    got = kp.csr_matvec(rp, ci, data, x)
    engine = "ref" if oracle.ref_spmv() is not None else "c"
    want = oracle.csr_matvec(rp, ci, data, x, engine=engine)
    assert np.array_equal(got, want)
    y1 = kp.csr_matvec(rp, ci, data, x[:, 0])
    assert y1.shape == (rp.shape[0] - 1,) and np.array_equal(y1, want[:, 0])


def test_csr_matvec_fuzz_rectangular_empty_rows(oracle, kpm_ctx):
    rng = np.random.default_rng(3)
    for _ in range(100):
        nrow, ncol = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        k = int(rng.integers(0, 5))
        dense = rng.standard_normal((nrow, ncol)) * (rng.random((nrow, ncol)) < 0.3)
        indptr = np.zeros(nrow + 1, dtype=np.int64)
        cols, vals = [], []
        for i in range(nrow):
            nzc = np.flatnonzero(dense[i])
            indptr[i + 1] = indptr[i] + nzc.size
            cols.append(nzc)
            vals.append(dense[i, nzc])
        idx = np.concatenate(cols).astype(np.int64)
        val = np.concatenate(vals)
        x = rng.standard_normal((ncol, k))
        got = kp.csr_matvec(indptr, idx, val, x)
        want = oracle.csr_matvec(indptr, idx, val, x, engine="c")
        assert got.shape == (nrow, k)
        assert np.array_equal(got, want)
    out = kp.csr_matvec(np.zeros(4, dtype=np.int64), np.zeros(0, dtype=np.int64),
                        np.zeros(0), np.ones((3, 2)))
    assert np.array_equal(out, np.zeros((3, 2)))


# ---------------------------------------------------------------- probes
@pytest.mark.parametrize("n,nz,c0", [(1000, 8, 0), (12345, 37, 5), (7, 3, 1)])
def test_device_rademacher_bitexact(kpm_ctx, n, nz, c0):
    ctx = kpm_ctx
    L = _lib.load()
    p = kp.make_probes(n, c0 + nz, "rademacher", seed=17)
    keys = p.column_slice(c0, c0 + nz).keys()
    ld = nz + 3
    buf = ctypes.c_void_p()
    _lib.check(L.kpm_device_alloc(ctx.handle, 8 * n * ld, ctypes.byref(buf)))
    _lib.check(L.kpm_probes_rademacher(ctx.handle, n, nz, _lib.ptr(keys), buf, ld, 2))
    got = _d2h(buf.value, (n, ld), ctx)[:, 2: 2 + nz]
    L.kpm_device_free(ctx.handle, buf)
    assert np.array_equal(got, p.columns[:, c0: c0 + nz])


def test_lazy_rademacher_run_equals_uploaded(kpm_ctx):
    g = kp.erdos_renyi(3000, 3e-3, seed=4)
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    lazy = kp.make_probes(g.n, 40, "rademacher", seed=9)
    host = kp.with_columns(lazy, kp.make_probes(g.n, 40, "rademacher", seed=9).columns)
    assert lazy.device_generated and not host.device_generated
    a = kp.dos_contrib(sop, lazy, 30)
    b = kp.dos_contrib(sop, host, 30)
    assert np.array_equal(a, b)


# ------------------------------------------------------ motif projection
def test_filter_probes_device_vs_reference(golden, golden_meta, kpm_ctx):
    n = int(golden["motif/n"])
    g = kp.GraphCSR(n=n, row_ptr=golden["motif/row_ptr"], col_idx=golden["motif/col_idx"],
                    weights=np.ones(golden["motif/col_idx"].size), is_weighted=False)
    insts = kp.detect_motifs(g, seed=3)
    p = kp.with_columns(kp.make_probes(n, 16, "rademacher", seed=3), golden["motif/probes"])
    filt, adj = kp.filter_probes(p, insts)
    assert np.max(np.abs(filt.columns - golden["motif/filtered"])) <= 1e-12
    assert {repr(k): v for k, v in adj.removed.items()} == golden_meta["motif"]["removed"]
    res = kp.kpm_dos(g, m_max=80, nz=16, probe_kind="rademacher", seed=3, bins=40,
                     filter_kinds=("open-twin", "closed-twin", "dangling-two-chain"))
    assert _normwise(res.moments.values, golden["motif/dos_values"]) <= 1e-9
    assert np.abs(res.histogram.masses - golden["motif/hist_masses"]).sum() <= 1e-6


# ------------------------------------------------------------ configs
def test_c1_config_vs_reference(golden, kpm_ctx):
    g = kp.erdos_renyi(10000, 1e-3, seed=0)
    for doubling in (True, False):
        res = kp.kpm_dos(g, m_max=200, nz=20, probe_kind="rademacher", seed=0, bins=100,
                         doubling=doubling)
        assert _normwise(res.moments.values, golden["c1/dos_values"]) <= 1e-9
        assert np.abs(res.histogram.masses - golden["c1/hist_masses"]).sum() <= 1e-6


def test_c2_shape_vs_reference(golden, kpm_ctx):
    g = kp.preferential_attachment(20000, 5, seed=1)
    mom, _ = kp.kpm_pdos(g, m_max=100, nz=64, probe_kind="rademacher", seed=1)
    rows = golden["c2s/rows"]
    assert np.max(np.abs(mom.values[rows] - golden["c2s/pdos_rows"])) <= 1e-12
    assert _normwise(mom.global_values, golden["c2s/global_values"]) <= 1e-9


# ------------------------------------------------ determinism / sharding
def test_runs_are_deterministic_and_batch_invariant(kpm_ctx):
    g = kp.preferential_attachment(5000, 5, seed=1)
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    p = kp.make_probes(g.n, 64, "rademacher", seed=1)
    a = kp.dos_contrib(sop, p, 60)
    b = kp.dos_contrib(sop, p, 60)
    assert np.array_equal(a, b)
    # per-probe reductions do not depend on how many probes share a launch:
    # the 1-vs-N-GPU probe-sharding identity
    for batch in (32, 8, 5):
        assert np.array_equal(kp.dos_contrib(sop, p, 60, batch=batch), a)
    d = kp.dos_contrib(sop, p, 60, doubling=False)
    assert np.array_equal(kp.dos_contrib(sop, p, 60, doubling=False, batch=7), d)


# ---------------------------------------------------------------- errors
def test_error_semantics(kpm_ctx):
    p3 = kp.build_csr([(0, 1), (1, 2)])
    op = kp.build_operator(p3, "laplacian")
    bad = kp.rescale_operator(op, (0.0, 1.5))
    probes = kp.make_probes(3, 2, "rademacher", seed=0)
    for doubling in (True, False):
        with pytest.raises(kp.RecurrenceBlowupError, match="margin"):
            kp.dos_moments(bad, probes, 600, doubling=doubling)
    with pytest.raises(kp.RecurrenceBlowupError, match="margin"):
        kp.pdos_moments(bad, probes, 600)
    sop = kp.scaled_operator_for(p3, "normalized-adjacency")
    with pytest.raises(ValueError, match="m_max"):
        kp.dos_moments(sop, probes, -1)
    with pytest.raises(ValueError, match="probe dimension"):
        kp.dos_moments(sop, kp.make_probes(4, 2, "rademacher"), 3)
    z = np.ones((3, 2))
    z[1] = 0.0
    zp = kp.ProbeMatrix(3, 2, "gaussian", 0, columns=z)
    with pytest.raises(ValueError, match="zero probe mass at node 1"):
        kp.pdos_moments(sop, zp, 4)
    raw = kp.pdos_moments(sop, zp, 4, normalized=False)
    assert np.all(raw.values[1] == 0.0)
    m0 = kp.dos_moments(sop, probes, 0)
    assert m0.values.shape == (1,) and m0.values[0] == pytest.approx(1.0, abs=1e-14)


# ------------------------------------------------------- hub (heavy) rows
@pytest.mark.parametrize("name", GRAPH_CASES)
@pytest.mark.parametrize("mode", [_lib.MODE_DOS_DIRECT, _lib.MODE_DOS_DOUBLING,
                                  _lib.MODE_LDOS])
def test_hub_path_bitexact(golden, kpm_ctx, monkeypatch, name, mode):
    """Force the column-sliced hub path (degree >= 3) and re-check the T
    blocks bit-for-bit and the moments against the reference."""
    monkeypatch.setenv("KPM_HEAVY_DEGREE", "3")
    g = _graph(golden, name)
    z = golden[f"{name}/probes"]
    dev = kp.DeviceGraph.from_csr(g.n, g.row_ptr, g.col_idx)
    steps = sorted(int(k.split("/T")[1]) for k in golden if k.startswith(f"{name}/T"))
    run = Run(dev, z.shape[1], mode, 2 * max(steps) + 2)
    run.set_probe_block(z, z.shape[1])
    done = 0
    for s in steps:
        run.advance(s - done)
        done = s
        ptr, ld, _ = run.block()
        t = _d2h(ptr, (g.n, ld), kpm_ctx)[:, : z.shape[1]]
        assert np.array_equal(t, golden[f"{name}/T{s}"]), (name, s)
    run.free()
    nz, seed, m_dos, m_pdos = golden[f"{name}/meta"].tolist()
    op = kp.NormalizedAdjacencyOperator(dev)
    sop = kp.rescale_operator(op, (-1.0, 1.0))
    probes = kp.ProbeMatrix(g.n, nz, "rademacher", seed, columns=z)
    if mode == _lib.MODE_LDOS:
        pd = kp.pdos_moments(sop, probes, m_pdos)
        assert np.max(np.abs(pd.values - golden[f"{name}/pdos_values"])) <= 1e-12
    else:
        mom = kp.dos_moments(sop, probes, m_dos, doubling=mode == _lib.MODE_DOS_DOUBLING)
        assert _normwise(mom.values, golden[f"{name}/dos_values"]) <= 1e-9


def test_hub_path_large_degree(oracle, kpm_ctx, monkeypatch):
    """A real hub (star + ER background, max degree ~6000) with 128 probes:
    hub rows take the sliced path at the default threshold; T_3 bit-exact."""
    rng = np.random.default_rng(0)
    n = 20000
    hub_nb = rng.choice(np.arange(1, n), 6000, replace=False)
    eu = rng.integers(0, n, 60000)
    ev = rng.integers(0, n, 60000)
    u = np.concatenate([np.zeros(6000, dtype=np.int64), eu])
    v = np.concatenate([hub_nb, ev])
    dev = kp.DeviceGraph.from_edges(n, u, v)
    assert dev.max_degree >= 6000
    rp, ci, dinv = dev.export()
    ci = ci.astype(np.int64)
    data = oracle.normadj_values(rp, ci, dinv)
    z = oracle.make_probes(n, 128, "rademacher", seed=1)
    run = Run(dev, 128, _lib.MODE_DOS_DIRECT, 6)
    run.set_probe_block(z, 128)
    run.advance(3)
    ptr, ld, _ = run.block()
    got = _d2h(ptr, (n, ld), kpm_ctx)[:, :128]
    run.free()
    assert np.array_equal(got, oracle.c_recurrence_block(rp, ci, data, z, 3, threads=8))
    op = kp.rescale_operator(kp.NormalizedAdjacencyOperator(dev), (-1.0, 1.0))
    c = kp.dos_contrib(op, kp.ProbeMatrix(n, 128, "rademacher", 1, columns=z), 20,
                       doubling=False)
    want = oracle.c_dos_contrib(rp, ci, data, z, 20, threads=8)
    assert _normwise(c, want) <= 1e-12


def _block_after(dev, z, mode, steps, ctx):
    run = Run(dev, z.shape[1], mode, 2 * steps + 2)
    run.set_probe_block(z, z.shape[1])
    run.advance(steps)
    ptr, ld, _ = run.block()
    t = _d2h(ptr, (dev.n, ld), ctx)[:, : z.shape[1]]
    run.free()
    return t


@pytest.mark.parametrize("P", [65, 100, 128])
@pytest.mark.parametrize("mode", [_lib.MODE_DOS_DIRECT, _lib.MODE_DOS_DOUBLING,
                                  _lib.MODE_LDOS])
def test_bulk_gather_path_bitexact(oracle, kpm_ctx, monkeypatch, P, mode):
    """The 4-column layout gathers neighbour rows with TMA bulk copies into a
    shared-memory ring (light_bulk): T blocks bit-identical to the oracle's
    restated recurrence and to the register-gather path, with and without the
    hot-row L2 policy."""
    g = kp.preferential_attachment(6000, 4, seed=9)
    dev = g.device()
    rp, ci, dinv = dev.export()
    ci = ci.astype(np.int64)
    z = oracle.make_probes(g.n, P, "rademacher", seed=P)
    want = oracle.c_recurrence_block(rp, ci, oracle.normadj_values(rp, ci, dinv), z, 4,
                                     threads=8)
    got = {}
    for bulk, hot in (("1", None), ("1", "4"), ("0", None)):
        monkeypatch.setenv("KPM_BULK", bulk)
        if hot:
            monkeypatch.setenv("KPM_HOT_DEGREE", hot)
        else:
            monkeypatch.delenv("KPM_HOT_DEGREE", raising=False)
        got[(bulk, hot)] = _block_after(dev, z, mode, 4, kpm_ctx)
    for key, t in got.items():
        assert np.array_equal(t, want), key


def test_bulk_gather_rmat_moments_match_register_path(kpm_ctx, monkeypatch):
    dev = kp.DeviceGraph.rmat(15, 16, seed=3)
    sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(dev), (-1.0, 1.0))
    z = kp.make_probes(dev.n, 128, "rademacher", seed=4)
    monkeypatch.setenv("KPM_BULK", "1")
    m1 = kp.dos_moments(sop, z, 40).values
    h1 = kp.pdos_moments(sop, z, 12).values
    monkeypatch.setenv("KPM_BULK", "0")
    m0 = kp.dos_moments(sop, z, 40).values
    h0 = kp.pdos_moments(sop, z, 12).values
    assert np.array_equal(m0, m1) and np.array_equal(h0, h1)


# ------------------------------------------------- device motif detection
def _inst_key(i):
    return (i.kind.value, tuple(i.nodes), i.eigenvalue, i.multiplicity,
            tuple(sorted((k, v) for vec in i.eigvecs for k, v in vec.items())))


def test_device_motif_scan_matches_reference(golden, golden_meta, kpm_ctx):
    n = int(golden["motif/n"])
    g = kp.GraphCSR(n=n, row_ptr=golden["motif/row_ptr"], col_idx=golden["motif/col_idx"],
                    weights=np.ones(golden["motif/col_idx"].size), is_weighted=False)
    dev = kp.detect_motifs(g, seed=3)
    assert type(dev).__name__ == "MotifSet"
    want = golden_meta["motif"]["instances"]
    assert len(dev) == len(want)
    for got, w in zip(dev, want):
        kind, nodes, lam, mult, vecs, _ = w
        assert got.kind.value == kind and list(got.nodes) == nodes
        assert got.eigenvalue == lam and got.multiplicity == mult
        for gv, wv in zip(got.eigvecs, vecs):
            assert sorted(gv.items()) == sorted((int(k), v) for k, v in wv)
    # array-backed filtering == the reference's filtered probes
    p = kp.with_columns(kp.make_probes(n, 16, "rademacher", seed=3), golden["motif/probes"])
    filt, adj = kp.filter_probes(p, dev)
    assert np.max(np.abs(filt.columns - golden["motif/filtered"])) <= 1e-12
    assert {repr(k): v for k, v in adj.removed.items()} == golden_meta["motif"]["removed"]


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("operator", ["normalized-adjacency", "adjacency", "laplacian",
                                      "normalized-laplacian"])
def test_device_motif_scan_matches_host(kpm_ctx, seed, operator):
    g = kp.testkit.motif_heavy(n_ba=4000, m=2, seed=seed, twin_pairs=300, stars=80)
    for kinds in (None, {kp.MotifKind.CLOSED_TWIN}, {kp.MotifKind.DANGLING_TWO_CHAIN}):
        dev = kp.detect_motifs(g, kinds=kinds, operator=operator)
        host = kp.detect_motifs(g, kinds=kinds, operator=operator, device=False)
        assert [_inst_key(i) for i in dev] == [_inst_key(i) for i in host]
        assert [(repr(i.detail), i._operator) for i in dev] == \
            [(repr(i.detail), i._operator) for i in host]
    # isolated nodes form one open-twin class; loops are excluded
    g2 = kp.build_csr([(0, 1), (0, 2), (3, 3), (4, 5)], n=9, allow_self_loops=True)
    assert [_inst_key(i) for i in kp.detect_motifs(g2)] == \
        [_inst_key(i) for i in kp.detect_motifs(g2, device=False)]


def test_filtered_probes_stay_on_device(golden, kpm_ctx):
    """Seeded Rademacher probes are generated, deflated and consumed in HBM;
    the result equals deflating the host block, and moments agree."""
    n = int(golden["motif/n"])
    g = kp.GraphCSR(n=n, row_ptr=golden["motif/row_ptr"], col_idx=golden["motif/col_idx"],
                    weights=np.ones(golden["motif/col_idx"].size), is_weighted=False)
    insts = kp.detect_motifs(g, seed=3)
    lazy = kp.make_probes(n, 16, "rademacher", seed=3)
    fd, adj = kp.filter_probes(lazy, insts)
    assert fd.device_block is not None and fd._columns is None
    fh, adj2 = kp.filter_probes(kp.with_columns(lazy, golden["motif/probes"]), insts)
    assert adj.removed == adj2.removed
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    md = kp.dos_moments(sop, fd, 60, effective_dim=n - adj.deflated_dim)
    mh = kp.dos_moments(sop, fh, 60, effective_dim=n - adj.deflated_dim)
    assert np.array_equal(md.values, mh.values)
    assert np.array_equal(fd.columns, fh.columns)
    half = fd.column_slice(4, 12)
    assert np.array_equal(half.columns, fh.columns[:, 4:12])


# Every light-row gather path of the step kernel, selected by environment
# (kpm_step.cu launch_c): TMA gather4 (default for ld % 4 == 0; the 4-column
# layout of the global modes as 64-column tiles, or whole rows with KPM_G4=2
# KPM_TILE=0), per-lane cp.async (KPM_G4=0), TMA bulk copies
# (KPM_LEAN=0) and register gathers (KPM_BULK=0); each with and without forced
# hub rows (cp.async hub pipeline), on the implicit normalized adjacency and on
# explicit values with shift/scale.  T blocks must be bit-identical to the
# oracle's restated recurrence (the reference's _row order, no FMA).
_PATHS = {
    "tiles": {},  # default: gather4, 4-column layouts as 64-column passes
    "tiles-unfused": {"KPM_FUSE_TILES": "0"},
    "g4": {"KPM_G4": "2", "KPM_TILE": "0"},
    "lean": {"KPM_G4": "0"},
    "bulk": {"KPM_G4": "0", "KPM_LEAN": "0"},
    "register": {"KPM_G4": "0", "KPM_LEAN": "0", "KPM_BULK": "0"},
}


@pytest.mark.parametrize("path", sorted(_PATHS))
@pytest.mark.parametrize("P", [4, 20, 30, 32, 36, 64, 100, 128])
@pytest.mark.parametrize("hubs", [False, True])
def test_light_paths_bitexact(oracle, kpm_ctx, monkeypatch, path, P, hubs):
    for k in ("KPM_G4", "KPM_TILE", "KPM_LEAN", "KPM_BULK", "KPM_HEAVY_DEGREE", "KPM_G4_HOT",
              "KPM_HOT_MB_G4", "KPM_FUSE_TILES"):
        monkeypatch.delenv(k, raising=False)
    for k, v in _PATHS[path].items():
        monkeypatch.setenv(k, v)
    if hubs:
        monkeypatch.setenv("KPM_HEAVY_DEGREE", "40")
    g = kp.preferential_attachment(3000, 3, seed=P)
    # 70 isolated vertices inserted at id 1500 and 300 appended: runs of empty rows, and
    # whole chunks of them (the streamed empty-chunk path)
    ins = lambda v: v + 70 * (v >= 1500)
    deg = np.diff(g.row_ptr)
    deg = np.concatenate([deg[:1500], np.zeros(70, np.int64), deg[1500:], np.zeros(300, np.int64)])
    n = g.n + 370
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = ins(g.col_idx.astype(np.int64))
    z = oracle.make_probes(n, P, "rademacher", seed=P + 1)
    dinv = oracle.dinv_of(rp)
    for mode in (_lib.MODE_DOS_DOUBLING, _lib.MODE_DOS_DIRECT, _lib.MODE_LDOS):
        dev = kp.DeviceGraph.from_csr(n, rp, ci)
        want = oracle.c_recurrence_block(rp, ci, oracle.normadj_values(rp, ci, dinv), z, 5,
                                         threads=8)
        assert np.array_equal(_block_after(dev, z, mode, 5, kpm_ctx), want), (path, mode)
    # explicit values (a shifted/scaled Laplacian-like operator)
    vals = -oracle.normadj_values(rp, ci, dinv)
    dev = kp.DeviceGraph.from_csr(n, rp, ci, values=vals, shift=0.25, scale=1.5)
    want = oracle.c_recurrence_block(rp, ci, vals, z, 5, shift=0.25, scale=1.5, threads=8)
    assert np.array_equal(_block_after(dev, z, _lib.MODE_DOS_DIRECT, 5, kpm_ctx), want), path
