"""Host-side logic of the package (no GPU): graph building, generators,
probes, histograms, motif detection / deflation bookkeeping, sharding maths.
Each is checked against the reference's own outputs (tests/golden) or the
oracle."""

import hashlib

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from conftest import GRAPH_CASES
from paper_1905_09758_b200 import motifs as M
from paper_1905_09758_b200.distributed import shard_range


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ graphs
def test_build_csr_small_graphs(golden):
    tri = kp.build_csr([(0, 1), (0, 2), (1, 2)])
    assert np.array_equal(tri.row_ptr, golden["triangle/row_ptr"])
    assert np.array_equal(tri.col_idx, golden["triangle/col_idx"])
    iso = kp.build_csr([(0, 1), (1, 2), (2, 3), (0, 3), (4, 5)], n=9)
    assert np.array_equal(iso.row_ptr, golden["isolated9/row_ptr"])
    assert np.array_equal(iso.degrees(), golden["isolated9/degrees"])


def test_build_csr_duplicate_semantics():
    # same-direction repeats sum weights (graph.py:130-160), unweighted flag
    g = kp.build_csr([(0, 1), (0, 1), (1, 2)])
    assert g.weights.tolist() == [2.0, 2.0, 1.0, 1.0] and not g.is_weighted
    # a restatement in the opposite direction with conflicting weight raises
    with pytest.raises(kp.GraphError, match="conflicting weights"):
        kp.build_csr([(0, 1), (0, 1), (1, 0)])
    # equal restatement is the same edge
    g2 = kp.build_csr([(0, 1), (1, 0)])
    assert g2.nnz == 2 and g2.weights.tolist() == [1.0, 1.0]
    with pytest.raises(kp.GraphError, match="self-loop"):
        kp.build_csr([(0, 0)])
    g3 = kp.build_csr([(0, 0), (0, 1)], allow_self_loops=True)
    assert g3.col_idx.tolist() == [0, 1, 0] and g3.num_edges == 2
    with pytest.raises(kp.GraphError, match="non-positive"):
        kp.build_csr([(0, 1, -1.0)])
    with pytest.raises(kp.GraphError, match="smaller than"):
        kp.build_csr([(0, 5)], n=3)
    e = kp.build_csr([], n=4)
    assert e.nnz == 0 and e.row_ptr.tolist() == [0] * 5


def test_er_generator_matches_reference(golden_meta):
    gens = golden_meta["generators"]
    for key, want in gens.items():
        if not key.startswith("er_"):
            continue
        _, n, p, s = key.split("_")
        g = kp.erdos_renyi(int(n), float(p), seed=int(s))
        assert g.nnz == want["nnz"], key
        assert _sha(g.row_ptr) == want["row_ptr"] and _sha(g.col_idx) == want["col_idx"], key


@pytest.mark.parametrize("key", ["ba_300_3_4", "ba_5000_5_1", "ba_20000_5_1",
                                 "ba_1000000_5_1", "ba_2000000_4_3"])
def test_ba_generator_matches_reference(golden_meta, key):
    """Native PCG64 replay (libkpm host code) reproduces the reference's BA
    graphs bit-for-bit, including the full C2 and C4 sizes."""
    want = golden_meta["generators"][key]
    _, n, m, s = key.split("_")
    g = kp.preferential_attachment(int(n), int(m), seed=int(s))
    assert g.nnz == want["nnz"]
    assert _sha(g.row_ptr) == want["row_ptr"] and _sha(g.col_idx) == want["col_idx"]


def test_ba_python_path_matches_reference(golden_meta):
    want = golden_meta["generators"]["ba_5000_5_1"]
    g = kp.preferential_attachment(5000, 5, seed=1, native=False)
    assert _sha(g.col_idx) == want["col_idx"]


def test_graph_cases_reproduced(golden):
    g = kp.erdos_renyi(200, 0.05, seed=3)
    assert np.array_equal(g.row_ptr, golden["er200/row_ptr"])
    g = kp.preferential_attachment(300, 3, seed=4)
    assert np.array_equal(g.col_idx, golden["ba300/col_idx"])


def test_host_operator_values_match_reference(golden):
    for name in GRAPH_CASES:
        n = int(golden[f"{name}/n"])
        rp, ci = golden[f"{name}/row_ptr"], golden[f"{name}/col_idx"]
        g = kp.GraphCSR(n=n, row_ptr=rp, col_idx=ci, weights=np.ones(ci.size),
                        is_weighted=False)
        op = kp.build_operator(g, "normalized-adjacency")
        assert op.implicit
        assert np.array_equal(op.data, golden[f"{name}/op_data"])


def test_explicit_operator_assembly_matches_reference(golden):
    g = kp.erdos_renyi(60, 0.1, seed=21)
    op = kp.build_operator(g, "laplacian")
    assert np.array_equal(op.indptr, golden["lap60/indptr"])
    assert np.array_equal(op.indices, golden["lap60/indices"])
    assert np.array_equal(op.data, golden["lap60/data"])


def test_normalized_range_is_analytic():
    g = kp.build_csr([(0, 1), (1, 2)])
    op = kp.build_operator(g, "normalized-adjacency")
    assert kp.estimate_spectral_range(op) == (-1.0, 1.0)
    sop = kp.rescale_operator(op, (-1.0, 1.0))
    assert sop.shift == 0.0 and sop.scale == 1.0
    with pytest.raises(ValueError, match="degenerate"):
        kp.rescale_operator(op, (1.0, 1.0))


# ------------------------------------------------------------------ probes
@pytest.mark.parametrize("kind", ["rademacher", "gaussian", "hadamard"])
def test_make_probes_match_reference(golden, kind):
    p = kp.make_probes(1000, 8, kind, seed=17)
    assert np.array_equal(p.columns, golden[f"probes/{kind}"])


def test_probe_slices_and_keys(golden):
    p = kp.make_probes(1000, 8, "rademacher", seed=17)
    assert p.device_generated
    s = p.column_slice(3, 6)
    assert s.device_generated and s.col_offset == 3
    assert np.array_equal(s.columns, golden["probes/rademacher"][:, 3:6])
    keys = s.keys()
    assert keys.dtype == np.uint64 and keys.shape == (6,)
    ss = np.random.SeedSequence(17).spawn(8)[4]
    assert np.array_equal(keys[2:4], np.random.Philox(ss).state["state"]["key"])
    assert kp.make_probes(6, 4, "standard-basis").columns.tolist() == \
        golden["probes/std_basis"].tolist()
    with pytest.raises(ValueError, match="nz <= n"):
        kp.make_probes(3, 4, "standard-basis")
    with pytest.raises(ValueError, match="nz must be"):
        kp.make_probes(3, 0)


def test_philox_bitstream_is_numpy_integers():
    """The device Rademacher kernel's bit rule: element i is bit 31 of the
    i-th 32-bit half of the Philox4x64 stream (low half first)."""
    ss = np.random.SeedSequence(5, spawn_key=(2,))
    want = np.random.Generator(np.random.Philox(ss)).integers(0, 2, size=64)
    raw = np.random.Philox(ss).random_raw(32)
    bits = np.empty(64, dtype=np.int64)
    bits[0::2] = (raw & np.uint64(0xFFFFFFFF)) >> np.uint64(31)
    bits[1::2] = raw >> np.uint64(63)
    assert np.array_equal(bits, want)


# --------------------------------------------------------------- density
@pytest.mark.parametrize("name", GRAPH_CASES)
def test_histogram_matches_reference(golden, name):
    mom = kp.ChebMoments("global", golden[f"{name}/dos_values"], kp.ScaleMap(0.0, 1.0), {})
    h = kp.histogram_from_moments(mom, bins=50)
    assert np.array_equal(h.edges, golden[f"{name}/hist_edges"])
    assert np.array_equal(h.masses, golden[f"{name}/hist_masses"])


def test_c1_histogram_from_reference_moments(golden):
    mom = kp.ChebMoments("global", golden["c1/dos_values"], kp.ScaleMap(0.0, 1.0), {})
    h = kp.histogram_from_moments(mom, bins=100)
    assert np.array_equal(h.masses, golden["c1/hist_masses"])


def test_jackson_properties():
    for m in (0, 1, 7, 500):
        assert kp.jackson_coefficients(m)[0] == 1.0
    j = kp.jackson_coefficients(100)
    assert np.all(np.diff(j) <= 1e-15) and j[-1] == pytest.approx(0.0, abs=1e-15)
    with pytest.raises(ValueError):
        kp.jackson_coefficients(-1)


# ---------------------------------------------------------------- motifs
def _motif_graph(golden):
    n = int(golden["motif/n"])
    return kp.GraphCSR(n=n, row_ptr=golden["motif/row_ptr"], col_idx=golden["motif/col_idx"],
                       weights=np.ones(golden["motif/col_idx"].size), is_weighted=False)


def test_detect_motifs_matches_reference(golden, golden_meta):
    g = _motif_graph(golden)
    insts = kp.detect_motifs(g, seed=3, device=False)
    want = golden_meta["motif"]["instances"]
    assert len(insts) == len(want)
    for got, w in zip(insts, want):
        kind, nodes, lam, mult, vecs, _ = w
        assert got.kind.value == kind and list(got.nodes) == nodes
        assert got.eigenvalue == lam and got.multiplicity == mult
        for gv, wv in zip(got.eigvecs, vecs):
            assert sorted(gv.items()) == sorted((int(k), v) for k, v in wv)


def test_deflation_bookkeeping_and_projection(golden, golden_meta, oracle):
    g = _motif_graph(golden)
    insts = kp.detect_motifs(g, seed=3, device=False)
    arrays, removed = M.deflation_vectors(insts, g.n)
    assert {repr(k): v for k, v in removed.items()} == golden_meta["motif"]["removed"]
    # grouping for the device kernel keeps every shared-support chain in order
    gp, vp, vi, vv = M.projection_groups(arrays)
    assert gp[0] == 0 and gp[-1] == len(arrays)
    assert vp[-1] == sum(a[0].size for a in arrays)
    # per-group serial projection == the reference's sequential loop
    cols = oracle.project_out(golden["motif/probes"], arrays)
    assert np.max(np.abs(cols - golden["motif/filtered"])) < 1e-12
    grouped = [(vi[vp[v]:vp[v + 1]], vv[vp[v]:vp[v + 1]]) for v in range(len(arrays))]
    cols2 = oracle.project_out(golden["motif/probes"], grouped)
    assert np.max(np.abs(cols2 - golden["motif/filtered"])) < 1e-12


def test_overlapping_claims_and_dependent_vectors():
    g = kp.build_csr([(0, 1), (0, 2), (0, 3)])
    twin = kp.detect_motifs(g, kinds={kp.MotifKind.OPEN_TWIN}, device=False)[0]
    fake = kp.MotifInstance(kind=kp.MotifKind.CUSTOM, nodes=(2, 3), eigenvalue=0.25,
                            eigvecs=({2: 1 / np.sqrt(2), 3: -1 / np.sqrt(2)},))
    _, removed = M.deflation_vectors([twin, fake], 4)
    assert removed == {0.0: 2}
    a = kp.MotifInstance(kind=kp.MotifKind.CUSTOM, nodes=(0, 1), eigenvalue=0.0,
                         eigvecs=({0: 1.0},))
    b = kp.MotifInstance(kind=kp.MotifKind.CUSTOM, nodes=(0, 1), eigenvalue=0.5,
                         eigvecs=({0: 1.0},))
    with pytest.raises(kp.MotifError, match="dependent"):
        M.deflation_vectors([a, b], 4)
    with pytest.raises(kp.MotifError, match="custom"):
        kp.detect_motifs(g, kinds={kp.MotifKind.CUSTOM}, device=False)
    p = kp.make_probes(5, 3, "rademacher", seed=1)
    out, adj = kp.filter_probes(p, [])
    assert out is p and adj.deflated_dim == 0


def test_c4_builder_shape():
    n, u, v = kp.testkit.motif_heavy_edges(n_ba=3000, m=4, seed=3, twin_pairs=300, stars=50)
    assert n == 3000 + 600 + 200
    assert np.all(u < v)
    g = kp.testkit.motif_heavy(n_ba=3000, m=4, seed=3, twin_pairs=300, stars=50)
    insts = kp.detect_motifs(g, kinds={kp.MotifKind.OPEN_TWIN}, device=False)
    r = sum(i.multiplicity for i in insts)
    assert r >= 300 + 100  # every pair leaves >= 1 vector, every star 2


# -------------------------------------------------------------- sharding
def test_shard_ranges_cover():
    for nz in (1, 7, 20, 128, 256):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(nz, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == nz
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_detected_fast_path_matches_general_path(golden, oracle):
    """The vectorised bookkeeping for detected instances yields exactly the
    general path's vectors (same order, same values) and groups."""
    g = _motif_graph(golden)
    insts = kp.detect_motifs(g, seed=3, device=False)
    fast = M._detected_deflation(insts, g.n)
    assert fast is not None
    (gp, vp, vi, vv), removed = fast
    arrays, removed2 = M.deflation_vectors(insts, g.n)
    assert removed == removed2
    assert vp[-1] == sum(a[0].size for a in arrays) and len(vp) - 1 == len(arrays)
    for v, (idx, val) in enumerate(arrays):
        assert np.array_equal(vi[vp[v]:vp[v + 1]], idx)
        assert np.array_equal(vv[vp[v]:vp[v + 1]], val)
    vecs = [(vi[vp[v]:vp[v + 1]], vv[vp[v]:vp[v + 1]]) for v in range(len(arrays))]
    cols = oracle.project_out(golden["motif/probes"], vecs)
    assert np.max(np.abs(cols - golden["motif/filtered"])) < 1e-12
    # custom instances take the general path
    custom = kp.MotifInstance(kind=kp.MotifKind.CUSTOM, nodes=(0, 2), eigenvalue=0.0,
                              eigvecs=({0: 1 / np.sqrt(2), 2: -1 / np.sqrt(2)},))
    assert M._detected_deflation(insts + [custom], g.n) is None


def test_lazy_instances_match_reference_fields(golden_meta, golden):
    g = _motif_graph(golden)
    insts = kp.detect_motifs(g, seed=3, device=False)
    for got, w in zip(insts, golden_meta["motif"]["instances"]):
        assert got.multiplicity == w[3]
        assert len(got.eigvecs) == w[3]


def test_device_scan_extraction_host_logic():
    """motifs._scan_classes / _merge_classes / _instances (the host half of
    device detection): runs of a stable (hash, row) sort become classes ordered
    by smallest member; runs with a failed exact check go to the collision
    fallback; heads that failed are dropped; singletons are not classes."""
    rng = np.random.default_rng(7)
    n_runs = 500
    runs = [np.sort(rng.choice(10_000, rng.integers(1, 5), replace=False)) for _ in range(n_runs)]
    collide_run, dead_run = 3, 4
    runs[collide_run] = np.array([1, 2, 3]) + 20_000
    runs[dead_run] = np.array([4, 5]) + 20_000
    rows = np.concatenate(runs).astype(np.int64)
    starts = np.cumsum([0] + [r.size for r in runs[:-1]])
    head = np.repeat(starts, [r.size for r in runs]).astype(np.int64)
    ok = np.ones(rows.size, np.int8)
    ok[starts[collide_run] + 1] = 0
    ok[starts[dead_run]] = 0
    ptr, members, fallback = M._scan_classes(rows, head, ok)
    assert len(fallback) == 1 and np.array_equal(fallback[0], runs[collide_run])
    want = sorted((r for i, r in enumerate(runs) if r.size >= 2 and i not in (collide_run, dead_run)),
                  key=lambda r: int(r[0]))
    got = [members[a:b] for a, b in zip(ptr[:-1], ptr[1:])]
    assert len(got) == len(want) and all(np.array_equal(a, b) for a, b in zip(got, want))
    extra = [np.array([20_001, 20_003])]
    ptr2, mem2 = M._merge_classes(ptr, members, extra)
    want2 = sorted(want + extra, key=lambda r: int(r[0]))
    assert [tuple(mem2[a:b]) for a, b in zip(ptr2[:-1], ptr2[1:])] == [tuple(r) for r in want2]
    op = kp.OperatorKind.NORMALIZED_ADJACENCY
    deg = rng.integers(1, 9, 30_000).astype(np.float64)
    cdeg = deg[mem2[ptr2[:-1]]]
    insts = M._instances(kp.MotifKind.CLOSED_TWIN, ptr2, mem2, (-1.0 / cdeg).tolist(),
                         [{"degree": d, "weight": 1.0} for d in cdeg.tolist()], op)
    for inst, r, d in zip(insts, want2, cdeg):
        ref = M._build_instance(kp.MotifKind.CLOSED_TWIN, r, {"degree": float(d), "weight": 1.0}, op)
        assert inst == ref and inst.multiplicity == ref.multiplicity and inst.auto
