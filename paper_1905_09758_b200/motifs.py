"""Motif detection (host) and motif-filtered probes (device projection).

API of netdos motifs.py: open twins, closed twins and dangling two-chains
carry known eigenvalues with locally supported eigenvectors; deflating those
eigenvectors out of the probe block (filter_probes) removes the spectral
spikes, which histogram_from_moments re-inserts.

* ``detect_motifs`` restates the reference's detection semantics (motifs.py:
  189-311) with vectorised numpy: exact neighbour-list signatures replace the
  hash-bucket + pairwise verification, producing the same classes.
* ``filter_probes`` keeps the reference's greedy claim order, orthonormality
  check and modified Gram-Schmidt (motifs.py:321-398) on the host, then runs
  the projection loop (motifs.py:400-403) as the batched sm_100a kernel K7:
  vectors are grouped into connected components of shared support, groups run
  in parallel and vectors inside a group keep their list order.
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import MotifError
from .operators import OperatorKind
from .probes import ProbeMatrix, with_columns


class MotifKind(str, Enum):
    OPEN_TWIN = "open-twin"
    CLOSED_TWIN = "closed-twin"
    DANGLING_TWO_CHAIN = "dangling-two-chain"
    CUSTOM = "custom"


_KIND_RANK = {MotifKind.OPEN_TWIN: 0, MotifKind.CLOSED_TWIN: 1,
              MotifKind.DANGLING_TWO_CHAIN: 2, MotifKind.CUSTOM: 3}


@dataclass
class MotifInstance:
    """A detected structure: nodes, eigenvalue, orthonormal sparse
    eigenvectors (dict node -> value) with H u = eigenvalue u."""

    kind: MotifKind
    nodes: tuple
    eigenvalue: float
    eigvecs: tuple
    detail: dict = field(default_factory=dict)

    @property
    def multiplicity(self) -> int:
        return len(self.eigvecs)


@dataclass
class FilterAdjustment:
    """Per-eigenvalue multiplicities removed by deflation."""

    removed: dict
    total_dim: int

    @property
    def deflated_dim(self) -> int:
        return int(sum(self.removed.values()))


def _helmert_rows(size):
    """Orthonormal basis of the sum-zero subspace of R^size (size-1 rows)."""
    rows = []
    for k in range(1, size):
        v = np.zeros(size)
        v[:k] = 1.0
        v[k] = -float(k)
        rows.append(v / np.sqrt(k * (k + 1.0)))
    return rows


def _twin_modes(kind, motif, degree, weight):
    kind = OperatorKind(kind)
    if motif is MotifKind.OPEN_TWIN:
        return {OperatorKind.ADJACENCY: 0.0, OperatorKind.NORMALIZED_ADJACENCY: 0.0,
                OperatorKind.LAPLACIAN: degree,
                OperatorKind.NORMALIZED_LAPLACIAN: 1.0}[kind]
    if degree <= 0:
        raise MotifError("closed twins require positive degree")
    return {OperatorKind.ADJACENCY: -weight,
            OperatorKind.NORMALIZED_ADJACENCY: -weight / degree,
            OperatorKind.LAPLACIAN: degree + weight,
            OperatorKind.NORMALIZED_LAPLACIAN: 1.0 + weight / degree}[kind]


def _chain_modes(kind):
    """(eigenvalue, x-amplitude, middle-amplitude) of the two chain modes."""
    kind = OperatorKind(kind)
    s2 = 1.0 / np.sqrt(2.0)
    if kind is OperatorKind.NORMALIZED_ADJACENCY:
        return ((s2, s2, s2), (-s2, s2, -s2))
    if kind is OperatorKind.ADJACENCY:
        return ((1.0, s2, s2), (-1.0, s2, -s2))
    if kind is OperatorKind.NORMALIZED_LAPLACIAN:
        return ((1.0 - s2, s2, s2), (1.0 + s2, s2, -s2))
    out = []
    for lam in ((3.0 - np.sqrt(5.0)) / 2.0, (3.0 + np.sqrt(5.0)) / 2.0):
        a, b = 1.0, 1.0 - lam
        nrm = np.hypot(a, b)
        out.append((lam, a / nrm, b / nrm))
    return tuple(out)


def motif_eigenvalue(inst: MotifInstance, kind) -> float:
    if inst.kind is MotifKind.CUSTOM:
        return inst.eigenvalue
    if inst.kind in (MotifKind.OPEN_TWIN, MotifKind.CLOSED_TWIN):
        return float(_twin_modes(kind, inst.kind, inst.detail["degree"],
                                 inst.detail.get("weight", 1.0)))
    return float(_chain_modes(kind)[inst.detail["mode"]][0])


def motif_eigenvectors(inst: MotifInstance, kind) -> tuple:
    kind = OperatorKind(kind)
    if inst.kind is MotifKind.CUSTOM:
        return inst.eigvecs
    if inst.kind in (MotifKind.OPEN_TWIN, MotifKind.CLOSED_TWIN):
        nodes = inst.nodes
        return tuple({nodes[i]: float(x) for i, x in enumerate(row) if x != 0.0}
                     for row in _helmert_rows(len(nodes)))
    _, alpha, beta = _chain_modes(kind)[inst.detail["mode"]]
    vecs = []
    for amp in _helmert_rows(len(inst.detail["chains"])):
        v = {}
        for a, (x, b) in zip(amp, inst.detail["chains"]):
            if a != 0.0:
                v[x] = float(a * alpha)
                v[b] = float(a * beta)
        vecs.append(v)
    return tuple(vecs)


def _build_instance(motif, nodes, detail, kind):
    inst = MotifInstance(kind=motif, nodes=tuple(int(x) for x in nodes), eigenvalue=0.0,
                         eigvecs=(), detail=detail)
    inst.eigenvalue = motif_eigenvalue(inst, kind)
    inst.eigvecs = motif_eigenvectors(inst, kind)
    return inst


# --------------------------------------------------------------- detection
def _row_ids(g):
    return np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))


def _signature_classes(g, members, row_ptr_of, cols_of, w_of):
    """Group `members` by exact (ids, weights) signature.  Candidates are
    keyed by (degree, two independent 64-bit label sums) and then verified
    element-wise, so collisions cannot merge different signatures."""
    if members.size < 2:
        return []
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([11, 0x5349474E])))
    lab1 = rng.integers(0, 2 ** 63, size=g.n, dtype=np.uint64)
    lab2 = rng.integers(0, 2 ** 63, size=g.n, dtype=np.uint64)
    starts, ends = row_ptr_of(members)
    deg = ends - starts
    idx = np.repeat(starts, deg) + (np.arange(deg.sum()) - np.repeat(np.cumsum(deg) - deg, deg))
    ids = cols_of(idx)
    wts = w_of(idx)
    seg = np.repeat(np.arange(members.size), deg)
    with np.errstate(over="ignore"):
        wbits = wts.view(np.uint64)
        h1 = np.zeros(members.size, dtype=np.uint64)
        h2 = np.zeros(members.size, dtype=np.uint64)
        np.add.at(h1, seg, lab1[ids] ^ wbits)
        np.add.at(h2, seg, lab2[ids] + wbits * np.uint64(0x9E3779B97F4A7C15))
    order = np.lexsort((members, h2, h1, deg))
    d_s, h1_s, h2_s, m_s = deg[order], h1[order], h2[order], members[order]
    brk = np.ones(order.size, dtype=bool)
    brk[1:] = (d_s[1:] != d_s[:-1]) | (h1_s[1:] != h1_s[:-1]) | (h2_s[1:] != h2_s[:-1])
    gid = np.cumsum(brk) - 1
    counts = np.bincount(gid)
    classes = []
    multi = np.flatnonzero(counts >= 2)
    if multi.size == 0:
        return []
    first = np.flatnonzero(brk)
    pos_in_order = {}
    for gi in multi.tolist():
        grp = m_s[first[gi]: first[gi] + counts[gi]]
        # exact verification against the group's first member
        sig = {}
        for node in grp.tolist():
            s0, s1 = row_ptr_of(np.array([node]))
            sl = slice(int(s0[0]), int(s1[0]))
            key = (cols_of(np.arange(sl.start, sl.stop)).tobytes(),
                   w_of(np.arange(sl.start, sl.stop)).tobytes())
            sig.setdefault(key, []).append(node)
        for mem in sig.values():
            if len(mem) >= 2:
                classes.append(sorted(mem))
    del pos_in_order
    return classes


def _open_twin_classes(g):
    """Nodes with identical neighbour lists and weights, no self-loop
    (motifs.py:197-210)."""
    rows = _row_ids(g)
    loop_nodes = np.unique(rows[g.col_idx == rows])
    ok = np.ones(g.n, dtype=bool)
    ok[loop_nodes] = False
    members = np.flatnonzero(ok)
    rp = g.row_ptr
    return _signature_classes(
        g, members, lambda m: (rp[m], rp[m + 1]),
        lambda idx: g.col_idx[idx], lambda idx: g.weights[idx])


def _closed_twin_classes(g):
    """Adjacent nodes whose neighbourhoods agree outside the pair
    (motifs.py:213-240): identical closed neighbourhoods N[i] = N(i) + {i}
    with one common pair weight.  Unit-weight graphs use the vectorised
    signature; weighted graphs take the reference's pairwise check."""
    rows = _row_ids(g)
    has_loop = np.zeros(g.n, dtype=bool)
    has_loop[rows[g.col_idx == rows]] = True
    deg = np.diff(g.row_ptr)
    if not g.is_weighted and (g.nnz == 0 or np.all(g.weights == 1.0)):
        # closed neighbourhood rows: insert i into its own sorted list
        members = np.flatnonzero(~has_loop & (deg > 0))
        if members.size < 2:
            return []
        cn_ptr = np.zeros(g.n + 1, dtype=np.int64)
        np.cumsum(deg + 1, out=cn_ptr[1:])
        cols = np.empty(cn_ptr[-1], dtype=np.int64)
        keyed = np.concatenate([rows * np.int64(g.n) + g.col_idx,
                                np.arange(g.n, dtype=np.int64) * np.int64(g.n + 1)])
        keyed.sort()
        cols[:] = keyed % np.int64(g.n)
        w = np.ones(cols.shape[0])
        classes = _signature_classes(g, members, lambda m: (cn_ptr[m], cn_ptr[m + 1]),
                                     lambda idx: cols[idx], lambda idx: w[idx])
        return [(c, 1.0) for c in classes]
    return _closed_twin_classes_weighted(g, has_loop)


def _closed_twin_classes_weighted(g, has_loop):
    out = []
    rows = _row_ids(g)
    cand = defaultdict(list)
    for i in range(g.n):
        if has_loop[i] or g.row_ptr[i + 1] == g.row_ptr[i]:
            continue
        sl = g.neighbor_slice(i)
        cand[tuple(sorted(set(g.col_idx[sl].tolist()) | {i}))].append(i)
    del rows
    for mem in cand.values():
        if len(mem) < 2:
            continue
        groups = []  # (rep, members, pair weight)
        for i in sorted(mem):
            for grp in groups:
                w = _closed_pair_weight(g, grp[0], i)
                if w is not None and (grp[2] is None or w == grp[2]):
                    grp[1].append(i)
                    grp[2] = w
                    break
            else:
                groups.append([i, [i], None])
        for _, members, w in groups:
            if len(members) >= 2:
                out.append((sorted(members), w))
    return out


def _closed_pair_weight(g, i, j):
    si, sj = g.neighbor_slice(i), g.neighbor_slice(j)
    ids_i, w_i = g.col_idx[si], g.weights[si]
    ids_j, w_j = g.col_idx[sj], g.weights[sj]
    pos = np.searchsorted(ids_i, j)
    if pos >= ids_i.shape[0] or ids_i[pos] != j:
        return None
    ki = ~np.isin(ids_i, [i, j])
    kj = ~np.isin(ids_j, [i, j])
    if np.array_equal(ids_i[ki], ids_j[kj]) and np.array_equal(w_i[ki], w_j[kj]):
        return float(w_i[pos])
    return None


def _dangling_chain_classes(g):
    """Pendant paths x - b - hub, >= 2 per hub (motifs.py:243-260)."""
    deg = np.diff(g.row_ptr)
    xs = np.flatnonzero(deg == 1)
    if xs.size == 0:
        return []
    b = g.col_idx[g.row_ptr[xs]]
    ok = (g.weights[g.row_ptr[xs]] == 1.0) & (deg[b] == 2)
    xs, b = xs[ok], b[ok]
    s = g.row_ptr[b]
    n0, n1 = g.col_idx[s], g.col_idx[s + 1]
    w_ok = (g.weights[s] == 1.0) & (g.weights[s + 1] == 1.0)
    other = np.where(n0 == xs, n1, n0)
    single = (n0 == xs) ^ (n1 == xs)  # exactly one neighbour of b differs from x
    keep = w_ok & single & (other != xs)
    xs, b, hub = xs[keep], b[keep], other[keep]
    hubs = defaultdict(list)
    for x, bb, h in zip(xs.tolist(), b.tolist(), hub.tolist()):
        hubs[h].append((x, bb))
    return [(h, sorted(ch)) for h, ch in sorted(hubs.items()) if len(ch) >= 2]


def detect_motifs(g, kinds=None, seed=0, operator=OperatorKind.NORMALIZED_ADJACENCY) -> list:
    """Motif instances with eigenpairs stated for ``operator`` (motifs.py:
    263-311); every class is exact (no false positives).  ``seed`` is kept for
    signature parity: classes are a function of the graph alone."""
    del seed
    from .graph import DeviceGraph
    if isinstance(g, DeviceGraph):
        g = g.to_host()
    if kinds is None:
        kinds = {MotifKind.OPEN_TWIN, MotifKind.CLOSED_TWIN, MotifKind.DANGLING_TWO_CHAIN}
    kinds = {MotifKind(k) for k in kinds}
    if MotifKind.CUSTOM in kinds:
        raise MotifError("custom instances are supplied by the caller, not detected")
    out = []
    degs = g.degrees()
    if MotifKind.OPEN_TWIN in kinds:
        for members in _open_twin_classes(g):
            out.append(_build_instance(MotifKind.OPEN_TWIN, members,
                                       {"degree": float(degs[members[0]])}, operator))
    if MotifKind.CLOSED_TWIN in kinds:
        for members, w in _closed_twin_classes(g):
            out.append(_build_instance(MotifKind.CLOSED_TWIN, members,
                                       {"degree": float(degs[members[0]]), "weight": w},
                                       operator))
    if MotifKind.DANGLING_TWO_CHAIN in kinds:
        for hub, chains in _dangling_chain_classes(g):
            nodes = tuple(sorted(x for ch in chains for x in ch))
            for mode in (0, 1):
                out.append(_build_instance(MotifKind.DANGLING_TWO_CHAIN, nodes,
                                           {"hub": hub, "chains": tuple(chains), "mode": mode},
                                           operator))
    out.sort(key=lambda t: (_KIND_RANK[t.kind], min(t.nodes), t.eigenvalue))
    return out


# ---------------------------------------------------------------- filtering
def _vector_arrays(vec):
    idx = np.fromiter(vec.keys(), dtype=np.int64, count=len(vec))
    val = np.fromiter(vec.values(), dtype=np.float64, count=len(vec))
    order = np.argsort(idx)
    return idx[order], val[order]


def _reorthonormalize(arrays, tol):
    """Modified Gram-Schmidt over sparse vectors (motifs.py:321-339)."""
    done = []
    for idx, val in arrays:
        comp = dict(zip(idx.tolist(), val.tolist()))
        for pidx, pval in done:
            c = sum(pval[i] * comp.get(node, 0.0) for i, node in enumerate(pidx.tolist()))
            if c != 0.0:
                for i, node in enumerate(pidx.tolist()):
                    comp[node] = comp.get(node, 0.0) - c * pval[i]
        nrm = np.sqrt(sum(v * v for v in comp.values()))
        if nrm < tol:
            raise MotifError("motif eigenvectors are linearly dependent; "
                             "cannot re-orthonormalize the deflation set")
        items = sorted(comp.items())
        done.append((np.array([k for k, _ in items], dtype=np.int64),
                     np.array([v / nrm for _, v in items])))
    return done


def deflation_vectors(instances, n, reorth_tol=1e-8):
    """Greedy claims + orthonormality check (motifs.py:342-398): returns
    (list of (idx, val) in projection order, removed multiplicities)."""
    order = sorted(instances, key=lambda t: (_KIND_RANK[t.kind], min(t.nodes), t.eigenvalue))
    claimed, claim_keys, accepted = set(), set(), []
    for inst in order:
        key = (inst.kind, inst.nodes)
        nodes = set(inst.nodes)
        if key in claim_keys:
            accepted.append(inst)
        elif not nodes & claimed:
            accepted.append(inst)
            claimed |= nodes
            claim_keys.add(key)
    arrays, owner = [], []
    removed = defaultdict(int)
    for iid, inst in enumerate(accepted):
        for vec in inst.eigvecs:
            arrays.append(_vector_arrays(vec))
            owner.append(iid)
        removed[float(inst.eigenvalue)] += inst.multiplicity
    if not arrays:
        return [], {}
    worst = max(abs(float(val @ val) - 1.0) for _, val in arrays)
    touch = defaultdict(list)
    for vid, (idx, _) in enumerate(arrays):
        for node in idx.tolist():
            touch[node].append(vid)
    checked = set()
    for vids in touch.values():
        if len(vids) < 2:
            continue
        for a in range(len(vids)):
            for b in range(a + 1, len(vids)):
                pair = (vids[a], vids[b])
                if owner[pair[0]] == owner[pair[1]] or pair in checked:
                    continue
                checked.add(pair)
                ia, va = arrays[pair[0]]
                ib, vb = arrays[pair[1]]
                common, pa, pb = np.intersect1d(ia, ib, return_indices=True)
                if common.size:
                    worst = max(worst, abs(float(va[pa] @ vb[pb])))
    if worst > reorth_tol:
        arrays = _reorthonormalize(arrays, reorth_tol)
    return arrays, dict(removed)


def projection_groups(arrays):
    """CSR arrays for kpm_filter_probes: vectors grouped into connected
    components of shared support (list order kept inside a group)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    nv = len(arrays)
    lens = np.fromiter((a[0].size for a in arrays), dtype=np.int64, count=nv)
    idx = np.concatenate([a[0] for a in arrays]) if nv else np.zeros(0, np.int64)
    val = np.concatenate([a[1] for a in arrays]) if nv else np.zeros(0)
    vid = np.repeat(np.arange(nv, dtype=np.int64), lens)
    nodes, node_id = np.unique(idx, return_inverse=True)
    m = coo_matrix((np.ones(idx.size), (vid, nv + node_id)),
                   shape=(nv + nodes.size, nv + nodes.size))
    _, label = connected_components(m, directed=False)
    vlab = label[:nv]
    order = np.lexsort((np.arange(nv), vlab))  # by group, then list order
    vlab_s = vlab[order]
    brk = np.ones(nv, dtype=bool)
    brk[1:] = vlab_s[1:] != vlab_s[:-1]
    group_ptr = np.append(np.flatnonzero(brk), nv).astype(np.int64)
    vstart = np.concatenate([[0], np.cumsum(lens)])
    new_lens = lens[order]
    vec_ptr = np.concatenate([[0], np.cumsum(new_lens)]).astype(np.int64)
    gather = np.concatenate([np.arange(vstart[v], vstart[v + 1]) for v in order]) \
        if nv else np.zeros(0, np.int64)
    return group_ptr, vec_ptr, np.ascontiguousarray(idx[gather]), np.ascontiguousarray(val[gather])


def project_probes(columns, arrays, ctx=None):
    """The projection loop (motifs.py:400-403) on the device: returns the
    deflated copy of ``columns``."""
    cols = np.array(columns, dtype=np.float64, order="C", copy=True)
    if not arrays:
        return cols
    ctx = ctx or _lib.Context.get()
    gp, vp, vi, vv = projection_groups(arrays)
    _lib.check(_lib.load().kpm_filter_probes(
        ctx.handle, cols.shape[0], cols.shape[1], _lib.ptr(cols), cols.shape[1],
        gp.shape[0] - 1, _lib.ptr(gp), _lib.ptr(vp), _lib.ptr(vi), _lib.ptr(vv)),
        "filter_probes")
    return cols


def filter_probes(probes: ProbeMatrix, instances, reorth_tol=1e-8):
    """Project motif eigenvectors out of every probe column (motifs.py:342-405);
    returns (deflated probes, FilterAdjustment)."""
    arrays, removed = deflation_vectors(instances, probes.n, reorth_tol)
    if not arrays:
        return probes, FilterAdjustment(removed={}, total_dim=probes.n)
    cols = project_probes(probes.columns, arrays)
    return with_columns(probes, cols), FilterAdjustment(removed=removed, total_dim=probes.n)
