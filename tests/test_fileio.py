"""Graph file ingest against fixtures written by the
reference's own parse_graph_file (tests/golden/make_fileio_golden.py).

CPU tests pin the host restatement (the path the device hands weighted /
unusual files back to); GPU tests run the device tokenizer + loader and
require the same graphs, id maps, exception types and messages."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1905_09758_b200 import fileio
from paper_1905_09758_b200.graph import build_csr

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = os.path.join(HERE, "golden", "files")
with open(os.path.join(HERE, "golden", "fileio.json")) as _fh:
    CASES = json.load(_fh)

# the cases whose result the device path must produce on its own
DEVICE_CASES = {
    "comments", "sparse_ids", "malformed_tokens", "malformed_int", "one_token",
    "mm_pattern", "mm_isolated", "mm_out_of_range", "mm_zero_index", "mm_count",
    "mm_hash_line", "mm_sniff_header", "empty", "only_comments", "negative_ids", "crlf",
    "both_directions", "self_loop", "self_loop_ok", "vt_ff_whitespace", "tab_comment",
    "random_small", "random_large", "random_mm",
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def check_case(name, fn):
    rec = CASES[name]
    path = os.path.join(FILES, rec["file"])
    if "error" in rec:
        with pytest.raises(Exception) as ei:
            fn(path, **rec["kwargs"])
        assert type(ei.value).__name__ == rec["error"], (name, ei.value)
        assert str(ei.value).replace(path, "{path}") == rec["message"]
        return
    g, ids = fn(path, **rec["kwargs"])
    assert g.n == rec["n"] and g.nnz == rec["nnz"], name
    assert bool(g.is_weighted) == rec["is_weighted"]
    assert g.num_edges == rec["num_edges"]
    assert sha(np.asarray(g.row_ptr, dtype=np.int64)) == rec["row_ptr"], name
    assert sha(np.asarray(g.col_idx, dtype=np.int64)) == rec["col_idx"], name
    assert sha(np.asarray(g.weights, dtype=np.float64)) == rec["weights"], name
    assert sha(np.asarray(ids, dtype=np.int64)) == rec["ids"], name
    if "row_ptr_v" in rec:
        assert np.asarray(g.row_ptr).tolist() == rec["row_ptr_v"]
        assert np.asarray(g.weights).tolist() == rec["weights_v"]
        assert np.asarray(ids).tolist() == rec["ids_v"]


def _host(path, allow_self_loops=False):
    return fileio._host_parse(path, None, allow_self_loops)


@pytest.mark.parametrize("name", sorted(CASES))
def test_host_restatement_matches_reference(name):
    check_case(name, _host)


def test_fixture_coverage():
    assert DEVICE_CASES <= set(CASES)
    errors = {r["error"] for r in CASES.values() if "error" in r}
    assert {"FileFormatError", "GraphError", "OverflowError", "UnicodeDecodeError"} <= errors


def test_write_edgelist_round_trip_host(tmp_path):
    g = build_csr([(0, 1, 2.0), (1, 2, 0.5), (0, 3, 1.0)])
    p = tmp_path / "g.txt"
    fileio.write_graph_edgelist(g, p)
    g2, _ = fileio._host_parse(str(p), None, False)
    assert np.array_equal(g.row_ptr, g2.row_ptr)
    assert np.array_equal(g.col_idx, g2.col_idx)
    assert np.array_equal(g.weights, g2.weights)
    assert p.read_text().splitlines()[0] == "# nodes 4 edges 3"


def test_unknown_format_rejected(tmp_path):
    p = tmp_path / "g.txt"
    p.write_text("0 1\n")
    with pytest.raises(ValueError, match="unknown graph format"):
        fileio._host_parse(str(p), "csv", False)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_device_parse_matches_reference(name, kpm_ctx):
    check_case(name, fileio.parse_graph_file)
    if name in DEVICE_CASES:
        assert fileio.last_ingest_path == "device", name


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["comments", "random_large", "random_mm", "self_loop_ok",
                                  "mm_isolated", "negative_ids"])
def test_load_graph_file_device_resident(name, kpm_ctx):
    rec = CASES[name]
    path = os.path.join(FILES, rec["file"])
    dev, ids = fileio.load_graph_file(path, **rec["kwargs"])
    rp, ci, di = dev.export()
    assert sha(rp) == rec["row_ptr"]
    assert sha(ci.astype(np.int64)) == rec["col_idx"]
    assert sha(np.asarray(ids, dtype=np.int64)) == rec["ids"]
    deg = np.diff(rp).astype(np.float64)
    ref = np.where(deg > 0, 1.0 / np.sqrt(np.where(deg > 0, deg, 1.0)), 0.0)
    assert np.array_equal(di, ref)


@pytest.mark.gpu
def test_load_graph_file_rejects_summed_weights(kpm_ctx):
    """same_dir.txt repeats 0-1 in the same direction: the reference's
    build_csr sums it to weight 2 with is_weighted=False, which the implicit
    unit-weight device graph cannot represent -> GraphError, never a silently
    different operator; parse_graph_file keeps the reference's weights."""
    from paper_1905_09758_b200.errors import GraphError
    path = os.path.join(FILES, "same_dir.txt")
    g, _ = fileio.parse_graph_file(path)
    assert not g.unit_weights and not g.is_weighted
    with pytest.raises(GraphError, match="non-unit edge weights"):
        fileio.load_graph_file(path)


@pytest.mark.gpu
def test_device_parse_large_rmat_text(tmp_path, kpm_ctx):
    """A 2^18-edge R-MAT edge list with comments, CRLF-free mixed whitespace
    and sparse ids: device ingest == host restatement, bit for bit."""
    from paper_1905_09758_b200.testkit import rmat
    g = rmat(16, 4, seed=5).to_host()
    u, v, _ = g.edge_list()
    rng = np.random.default_rng(0)
    perm = rng.permutation(g.n).astype(np.int64) * 7 - 1000   # sparse, some negative
    flip = rng.random(u.shape[0]) < 0.5
    a, b = np.where(flip, perm[v], perm[u]), np.where(flip, perm[u], perm[v])
    lines = [f"{x}\t{y}" if k % 3 else f" {x}  {y} " for k, (x, y) in
             enumerate(zip(a.tolist(), b.tolist()))]
    for k in range(0, len(lines), 1000):
        lines[k] = "# block %d\n" % k + lines[k]
    p = tmp_path / "rmat.txt"
    p.write_text("\n".join(lines) + "\n")
    gd, ids = fileio.parse_graph_file(str(p))
    assert fileio.last_ingest_path == "device"
    gh, idh = fileio._host_parse(str(p), None, False)
    assert np.array_equal(ids, idh)
    assert np.array_equal(gd.row_ptr, gh.row_ptr)
    assert np.array_equal(gd.col_idx, gh.col_idx)
    assert gd.n == gh.n and not gh.is_weighted


@pytest.mark.gpu
def test_device_parse_then_kpm(kpm_ctx):
    """The ingested device graph drives the moment pipeline directly."""
    import paper_1905_09758_b200 as kp
    rec = CASES["random_large"]
    path = os.path.join(FILES, rec["file"])
    dev, _ = kp.load_graph_file(path)
    g, _ = fileio._host_parse(path, None, False)
    sop_d = kp.rescale_operator(kp.NormalizedAdjacencyOperator(dev), (-1.0, 1.0))
    sop_h = kp.rescale_operator(kp.NormalizedAdjacencyOperator(g), (-1.0, 1.0))
    z = kp.make_probes(g.n, 8, "rademacher", seed=1)
    m1 = kp.dos_moments(sop_d, z, 40)
    m2 = kp.dos_moments(sop_h, z, 40)
    assert np.array_equal(m1.values, m2.values)
