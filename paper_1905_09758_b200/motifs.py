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


class MotifInstance:
    """A detected structure: nodes, eigenvalue, orthonormal sparse
    eigenvectors (dict node -> value) with H u = eigenvalue u (motifs.py:
    52-67 fields).  Detected instances build their eigenvector dicts lazily
    (``operator`` set): filter_probes reads the class structure directly, so
    C4's ~7.6e5 vectors never become Python dicts unless a caller asks."""

    __slots__ = ("kind", "nodes", "eigenvalue", "_eigvecs", "detail", "_operator")

    def __init__(self, kind, nodes, eigenvalue, eigvecs=None, detail=None, operator=None):
        self.kind = MotifKind(kind)
        self.nodes = tuple(nodes)
        self.eigenvalue = eigenvalue
        self._eigvecs = None if eigvecs is None else tuple(eigvecs)
        self.detail = {} if detail is None else detail
        self._operator = operator

    @property
    def eigvecs(self) -> tuple:
        if self._eigvecs is None:
            self._eigvecs = (motif_eigenvectors(self, self._operator)
                             if self._operator is not None else ())
        return self._eigvecs

    @eigvecs.setter
    def eigvecs(self, value):
        self._eigvecs = tuple(value)
        self._operator = None

    @property
    def auto(self) -> bool:
        """True for an untouched detected instance (structure known)."""
        return self._operator is not None and self.kind is not MotifKind.CUSTOM

    @property
    def multiplicity(self) -> int:
        if self.auto and self._eigvecs is None:
            if self.kind is MotifKind.DANGLING_TWO_CHAIN:
                return len(self.detail["chains"]) - 1
            return len(self.nodes) - 1
        return len(self.eigvecs)

    def __repr__(self):
        return (f"MotifInstance(kind={self.kind.value!r}, nodes={self.nodes}, "
                f"eigenvalue={self.eigenvalue!r}, detail={self.detail!r})")

    def __eq__(self, other):
        return (isinstance(other, MotifInstance) and self.kind is other.kind
                and self.nodes == other.nodes and self.eigenvalue == other.eigenvalue
                and self.eigvecs == other.eigvecs and self.detail == other.detail)


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
                         detail=detail, operator=OperatorKind(kind))
    inst.eigenvalue = motif_eigenvalue(inst, kind)
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
    multi = np.flatnonzero(counts >= 2)
    if multi.size == 0:
        return []
    first = np.flatnonzero(brk)
    # exact verification, vectorised: every member of a candidate group is
    # compared entry by entry with the group's first member
    in_multi = counts[gid] >= 2
    mem = m_s[in_multi]
    rep = m_s[first[gid[in_multi]]]
    ms, me = row_ptr_of(mem)
    rs, _ = row_ptr_of(rep)
    dd = me - ms
    tot = int(dd.sum())
    offs = np.arange(tot) - np.repeat(np.cumsum(dd) - dd, dd)
    im = np.repeat(ms, dd) + offs
    ir = np.repeat(rs, dd) + offs
    eq = (cols_of(im) == cols_of(ir)) & (w_of(im) == w_of(ir))
    bad_entry = np.repeat(np.arange(mem.size), dd)[~eq]
    ok = np.ones(mem.size, dtype=bool)
    ok[bad_entry] = False
    gm = gid[in_multi]
    bad_groups = np.unique(gm[~ok])
    classes = []
    good = ~np.isin(gm, bad_groups)
    gsel, msel = gm[good], mem[good]
    if gsel.size:
        cut = np.flatnonzero(np.diff(gsel)) + 1
        for grp in np.split(msel, cut):
            if grp.size >= 2:
                classes.append(sorted(grp.tolist()))
    # hash collisions (different lists, same key): exact regrouping
    for gi in bad_groups.tolist():
        grp = m_s[first[gi]: first[gi] + counts[gi]]
        sig = {}
        for node in grp.tolist():
            s0, s1 = row_ptr_of(np.array([node]))
            ar = np.arange(int(s0[0]), int(s1[0]))
            sig.setdefault((cols_of(ar).tobytes(), w_of(ar).tobytes()), []).append(node)
        for members_ in sig.values():
            if len(members_) >= 2:
                classes.append(sorted(members_))
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


def detect_motifs(g, kinds=None, seed=0, operator=OperatorKind.NORMALIZED_ADJACENCY,
                  device=True) -> list:
    """Motif instances with eigenpairs stated for ``operator`` (motifs.py:
    263-311); every class is exact (no false positives).  ``seed`` is kept for
    signature parity: classes are a function of the graph alone.  Unit-weight
    graphs are scanned on the B200 (csrc/kpm_motif.cu); ``device=False`` (or a
    weighted graph) runs the vectorised host restatement."""
    del seed
    from .graph import DeviceGraph
    if kinds is None:
        kinds = {MotifKind.OPEN_TWIN, MotifKind.CLOSED_TWIN, MotifKind.DANGLING_TWO_CHAIN}
    kinds = {MotifKind(k) for k in kinds}
    if MotifKind.CUSTOM in kinds:
        raise MotifError("custom instances are supplied by the caller, not detected")
    operator = OperatorKind(operator)
    if isinstance(g, DeviceGraph) or (device and g.unit_weights):
        return _detect_device(g, kinds, operator)
    return _detect_host(g, kinds, operator)


def _detect_host(g, kinds, operator) -> list:
    """General (weighted-graph) detection on the host."""
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


class MotifSet(list):
    """detect_motifs' result: the MotifInstance list of the reference API,
    plus the class arrays it was built from (``arrays``), which filter_probes
    uses directly while the list is unmodified."""

    def __init__(self, items, arrays, n):
        super().__init__(items)
        self.arrays = arrays
        self.n = n
        self._orig = tuple(items)

    def pristine(self) -> bool:
        return len(self) == len(self._orig) and all(a is b for a, b in zip(self, self._orig))


def _scan_classes(rows, head, ok):
    """Classes from a device signature scan: runs of equal signature whose
    members all matched the run head exactly, as (ptr, members) CSR arrays
    ordered by smallest member (rows of a run are ascending: the device sort
    is stable over row order); runs holding a mismatch (hash collision) come
    back as a list of row arrays for exact regrouping."""
    n = rows.shape[0]
    if n == 0:
        return np.zeros(1, np.int64), np.zeros(0, np.int64), []
    starts = np.flatnonzero(head == np.arange(n))
    lens = np.diff(np.append(starts, n))
    head_ok = ok[starts].astype(bool)
    bad = np.logical_or.reduceat(ok == 0, starts)
    keep = head_ok & ~bad & (lens >= 2)
    collide = head_ok & bad
    fallback = [rows[s:s + l] for s, l in zip(starts[collide].tolist(), lens[collide].tolist())]
    ks, kl = starts[keep], lens[keep]
    order = np.argsort(rows[ks], kind="stable")
    ks, kl = ks[order], kl[order]
    ptr = np.zeros(ks.size + 1, np.int64)
    np.cumsum(kl, out=ptr[1:])
    members = rows[np.repeat(ks - ptr[:-1], kl) + np.arange(ptr[-1])]
    return ptr, members, fallback


def _merge_classes(ptr, members, extra):
    """(ptr, members) plus extra class arrays, re-ordered by smallest member."""
    if not extra:
        return ptr, members
    classes = [members[a:b] for a, b in zip(ptr[:-1].tolist(), ptr[1:].tolist())] + extra
    classes.sort(key=lambda c: int(c[0]))
    sizes = np.fromiter((c.size for c in classes), np.int64, len(classes))
    ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return ptr, np.concatenate(classes).astype(np.int64)


def _instances(kind, ptr, members, eig, details, operator):
    """MotifInstance objects for detected classes without the per-object
    conversions of __init__ (kind, nodes and values are already canonical)."""
    ml, pl = members.tolist(), ptr.tolist()
    new = object.__new__
    out = []
    append = out.append
    for i, (lam, det) in enumerate(zip(eig, details)):
        inst = new(MotifInstance)
        inst.kind = kind
        inst.nodes = tuple(ml[pl[i]:pl[i + 1]])
        inst.eigenvalue = lam
        inst._eigvecs = None
        inst.detail = det
        inst._operator = operator
        append(inst)
    return out


def _detect_device(g, kinds, operator) -> "MotifSet":
    """Unit-weight detection: device signature scan (csrc/kpm_motif.cu) +
    O(n) host extraction; instances are created in the reference's order."""
    import ctypes

    from .graph import DeviceGraph
    dev = g if isinstance(g, DeviceGraph) else g.device()
    n = dev.n
    orow, crow = np.empty(n, np.int64), np.empty(n, np.int64)
    ohead, chead = np.empty(n, np.int64), np.empty(n, np.int64)
    ook, cok = np.empty(n, np.int8), np.empty(n, np.int8)
    hub, mid = np.empty(n, np.int64), np.empty(n, np.int64)
    _lib.check(_lib.load().kpm_motif_scan(
        dev.handle, _lib.ptr(orow), _lib.ptr(ook), _lib.ptr(ohead), _lib.ptr(crow),
        _lib.ptr(cok), _lib.ptr(chead), _lib.ptr(hub), _lib.ptr(mid)), "motif_scan")
    del ctypes
    rp = None
    deg = None

    def _rowptr():
        nonlocal rp, deg
        if rp is None:
            rp = dev.export()[0] if isinstance(g, DeviceGraph) else g.row_ptr
            deg = np.diff(rp).astype(np.float64)
        return rp

    def _exact(groups, closed):
        """Hash-collision runs: exact regrouping on the host (rare)."""
        hg = g if not isinstance(g, DeviceGraph) else g.to_host()
        out = []
        for rows in groups:
            sig = {}
            for i in sorted(rows.tolist()):
                nb = set(hg.neighbors(i).tolist())
                key = tuple(sorted(nb | {i})) if closed else tuple(sorted(nb))
                sig.setdefault(key, []).append(i)
            out.extend(np.asarray(m, dtype=np.int64) for m in sig.values() if len(m) >= 2)
        return out

    arrays = {"operator": operator}
    items = []
    _rowptr()
    for kind, rows, head, ok, closed in ((MotifKind.OPEN_TWIN, orow, ohead, ook, False),
                                         (MotifKind.CLOSED_TWIN, crow, chead, cok, True)):
        if kind not in kinds:
            arrays[kind] = (np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
            continue
        ptr, members, fallback = _scan_classes(rows, head, ok)
        ptr, members = _merge_classes(ptr, members, _exact(fallback, closed))
        cdeg = deg[members[ptr[:-1]]]
        arrays[kind] = (ptr, members, cdeg)
        dl = cdeg.tolist()
        if closed:
            if cdeg.size and cdeg.min() <= 0:
                raise MotifError("closed twins require positive degree")
            eig = [float(_twin_modes(operator, kind, d, 1.0)) for d in dl] \
                if operator is not OperatorKind.NORMALIZED_ADJACENCY else (-1.0 / cdeg).tolist()
            details = [{"degree": d, "weight": 1.0} for d in dl]
        else:
            eig = [float(_twin_modes(operator, kind, d, 1.0)) for d in dl] \
                if operator is OperatorKind.LAPLACIAN else \
                [float(_twin_modes(operator, kind, 1.0, 1.0))] * len(dl)
            details = [{"degree": d} for d in dl]
        items.extend(_instances(kind, ptr, members, eig, details, operator))
    if MotifKind.DANGLING_TWO_CHAIN in kinds:
        xs = np.flatnonzero(hub >= 0)
        order = np.argsort(hub[xs], kind="stable")
        xs = xs[order]
        hs, bs = hub[xs], mid[xs]
        if xs.size:
            cut = np.flatnonzero(np.diff(hs)) + 1
            starts = np.concatenate([[0], cut])
            ends = np.concatenate([cut, [xs.size]])
        else:
            starts = ends = np.zeros(0, np.int64)
        modes = _chain_modes(operator)
        chain_groups = []
        for s, e in zip(starts.tolist(), ends.tolist()):
            if e - s < 2:
                continue
            chains = tuple(zip(xs[s:e].tolist(), bs[s:e].tolist()))
            chain_groups.append((int(hs[s]), chains))
        chain_groups.sort(key=lambda t: min(min(x, b) for x, b in t[1]))
        arrays[MotifKind.DANGLING_TWO_CHAIN] = chain_groups
        for h, chains in chain_groups:
            nodes = tuple(sorted(v for ch in chains for v in ch))
            mode_order = sorted((0, 1), key=lambda mo: modes[mo][0])
            for mo in mode_order:
                inst = MotifInstance(MotifKind.DANGLING_TWO_CHAIN, nodes, float(modes[mo][0]),
                                     detail={"hub": h, "chains": chains, "mode": mo},
                                     operator=operator)
                items.append(inst)
    else:
        arrays[MotifKind.DANGLING_TWO_CHAIN] = []
    # reference order (rank, min node, eigenvalue): kinds already in rank
    # order, classes sorted by their smallest member
    return MotifSet(items, arrays, n)


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


def _detected_deflation(instances, n, reorth_tol=1e-8):
    """Vectorised filter_probes bookkeeping for untouched detected instances
    (the C4 case: ~6e5 classes).  Same greedy claim order, same vectors, same
    projection order as motifs.py:342-403, without per-vector Python objects.
    Returns ((group_ptr, vec_ptr, vec_idx, vec_val), removed) or None when
    the general path is needed (custom instances, overlaps inside a kind,
    non-orthonormal sets)."""
    if not instances or not all(getattr(i, "auto", False) for i in instances):
        return None
    m = len(instances)
    rank = np.fromiter((_KIND_RANK[i.kind] for i in instances), np.int64, m)
    mn = np.fromiter((i.nodes[0] for i in instances), np.int64, m)  # nodes sorted
    ev = np.fromiter((i.eigenvalue for i in instances), np.float64, m)
    order = np.lexsort((ev, mn, rank))  # stable, = sorted(key=(rank, min, ev))
    claimed = np.zeros(n, dtype=bool)
    accepted = np.zeros(m, dtype=bool)
    for rk in (0, 1, 2):
        sel = order[rank[order] == rk]
        if sel.size == 0:
            continue
        nodes_all = np.concatenate([np.asarray(instances[i].nodes, dtype=np.int64)
                                    for i in sel])
        lens = np.fromiter((len(instances[i].nodes) for i in sel), np.int64, sel.size)
        owner = np.repeat(np.arange(sel.size), lens)
        if rk == 2:  # the two modes of one hub share nodes; hubs must not
            hub = np.fromiter((instances[i].detail["hub"] for i in sel), np.int64, sel.size)
            pairs = np.unique(np.stack([hub[owner], nodes_all]), axis=1)
            if np.unique(pairs[1]).size != pairs.shape[1]:
                return None
        elif np.unique(nodes_all).size != nodes_all.size:
            return None  # overlapping classes inside a kind: general path
        bad = np.zeros(sel.size, dtype=bool)
        np.logical_or.at(bad, owner, claimed[nodes_all])
        accepted[sel[~bad]] = True
        claimed[nodes_all[~bad[owner]]] = True
    acc = order[accepted[order]]
    if acc.size == 0:
        return None
    removed = defaultdict(int)
    for i in acc.tolist():
        removed[float(instances[i].eigenvalue)] += instances[i].multiplicity

    # -- vectors (instance position p in acc order, Helmert index k) -------
    blocks = []  # (pos array, k, idx 2-D, val 2-D)
    twin_pos = [p for p, i in enumerate(acc.tolist()) if instances[i].kind is not
                MotifKind.DANGLING_TWO_CHAIN]
    by_size = defaultdict(list)
    for p in twin_pos:
        by_size[len(instances[acc[p]].nodes)].append(p)
    for s, plist in by_size.items():
        pos = np.asarray(plist, dtype=np.int64)
        nodes2d = np.asarray([instances[acc[p]].nodes for p in plist], dtype=np.int64)
        for k in range(1, s):
            nrm = np.sqrt(k * (k + 1.0))
            vals = np.empty(k + 1)
            vals[:k] = 1.0 / nrm
            vals[k] = -float(k) / nrm
            blocks.append((pos, k, nodes2d[:, : k + 1], np.broadcast_to(vals, (pos.size, k + 1))))
    chain_pos = [p for p, i in enumerate(acc.tolist()) if instances[i].kind is
                 MotifKind.DANGLING_TWO_CHAIN]
    for p in chain_pos:
        inst = instances[acc[p]]
        _, alpha, beta = _chain_modes(inst._operator)[inst.detail["mode"]]
        chains = inst.detail["chains"]
        for k, amp in enumerate(_helmert_rows(len(chains)), start=1):
            ent = {}
            for a, (x, b) in zip(amp, chains):
                if a != 0.0:
                    ent[x] = float(a * alpha)
                    ent[b] = float(a * beta)
            ks = sorted(ent)
            blocks.append((np.array([p]), k, np.array([ks], dtype=np.int64),
                           np.array([[ent[q] for q in ks]])))
    # orthonormality check (motifs.py:377-398): norms, and the only
    # cross-instance overlaps left -- two chain modes of one hub
    worst = 0.0
    for _, _, _, val in blocks:
        worst = max(worst, float(np.max(np.abs(np.einsum("ij,ij->i", val, val) - 1.0))))
    if chain_pos:
        per_hub = defaultdict(list)
        for p in chain_pos:
            per_hub[instances[acc[p]].detail["hub"]].append(p)
        vec_of = defaultdict(list)
        chain_set = set(chain_pos)
        for pos, k, idx, val in blocks:
            if pos.size == 1 and int(pos[0]) in chain_set:
                vec_of[int(pos[0])].append((idx[0], val[0]))
        for ps in per_hub.values():
            for a in range(len(ps)):
                for b in range(a + 1, len(ps)):
                    for ia, va in vec_of[ps[a]]:
                        for ib, vb in vec_of[ps[b]]:
                            _, pa, pb = np.intersect1d(ia, ib, return_indices=True)
                            if pa.size:
                                worst = max(worst, abs(float(va[pa] @ vb[pb])))
    if worst > reorth_tol:
        return None
    # -- CSR in projection order, groups = instances (chain modes of a hub
    # merged) ----------------------------------------------------------------
    vpos = np.concatenate([b[0] for b in blocks])
    vk = np.concatenate([np.full(b[0].size, b[1]) for b in blocks])
    vlen = np.concatenate([np.full(b[0].size, b[2].shape[1]) for b in blocks])
    eidx = np.concatenate([b[2].reshape(-1) for b in blocks])
    evals = np.concatenate([np.ascontiguousarray(b[3]).reshape(-1) for b in blocks])
    estart = np.concatenate([[0], np.cumsum(vlen)[:-1]])
    vorder = np.lexsort((vk, vpos))
    lens_o = vlen[vorder]
    vec_ptr = np.concatenate([[0], np.cumsum(lens_o)]).astype(np.int64)
    gather = (np.repeat(estart[vorder], lens_o) +
              (np.arange(int(lens_o.sum())) - np.repeat(vec_ptr[:-1], lens_o)))
    vec_idx = np.ascontiguousarray(eidx[gather])
    vec_val = np.ascontiguousarray(evals[gather])
    gkey = np.array([instances[i].detail["hub"] + n if instances[i].kind is
                     MotifKind.DANGLING_TWO_CHAIN else -1 - p
                     for p, i in enumerate(acc.tolist())], dtype=np.int64)
    vg = gkey[vpos[vorder]]
    brk = np.ones(vg.size, dtype=bool)
    brk[1:] = vg[1:] != vg[:-1]
    group_ptr = np.append(np.flatnonzero(brk), vg.size).astype(np.int64)
    return (group_ptr, vec_ptr, vec_idx, vec_val), dict(removed)


def _helmert_block(pos, nodes2d):
    """Helmert vectors of equal-size classes (rows of nodes2d, sorted members):
    yields (pos, k, idx2d, val2d) for k = 1..s-1 (motifs.py:71-79 values)."""
    s = nodes2d.shape[1]
    for k in range(1, s):
        nrm = np.sqrt(k * (k + 1.0))
        vals = np.empty(k + 1)
        vals[:k] = 1.0 / nrm
        vals[k] = -float(k) / nrm
        yield pos, k, nodes2d[:, : k + 1], np.broadcast_to(vals, (pos.size, k + 1))


def _deflation_from_arrays(arrays, n, reorth_tol=1e-8):
    """filter_probes bookkeeping straight from detect_motifs' class arrays:
    greedy claims (open twins, then closed twins, then chain hubs -- classes
    of one kind are disjoint), Helmert / chain vectors, per-class groups."""
    op = arrays["operator"]
    claimed = np.zeros(n, dtype=bool)
    blocks, gkeys, removed = [], [], defaultdict(int)
    next_pos = 0
    for kind in (MotifKind.OPEN_TWIN, MotifKind.CLOSED_TWIN):
        ptr, members, cdeg = arrays[kind]
        ncls = ptr.size - 1
        if ncls <= 0:
            continue
        sizes = np.diff(ptr)
        owner = np.repeat(np.arange(ncls), sizes)
        bad = np.zeros(ncls, dtype=bool)
        np.logical_or.at(bad, owner, claimed[members])
        claimed[members[~bad[owner]]] = True
        acc = np.flatnonzero(~bad)
        pos = next_pos + np.arange(acc.size)
        next_pos += acc.size
        udeg, dinv_ = np.unique(cdeg[acc], return_inverse=True)
        ev = np.array([_twin_modes(op, kind, float(d), 1.0) for d in udeg.tolist()])[dinv_]
        for sz in np.unique(sizes[acc]).tolist():
            sel = sizes[acc] == sz
            starts = ptr[acc[sel]]
            nodes2d = members[starts[:, None] + np.arange(sz)[None, :]]
            blocks.extend(_helmert_block(pos[sel], nodes2d))
        gkeys.append(pos)
        if acc.size:
            vals, inv = np.unique(ev, return_inverse=True)
            mult = np.bincount(inv, weights=sizes[acc] - 1)
            for v, m in zip(vals.tolist(), mult.tolist()):
                removed[float(v)] += int(m)
    modes = _chain_modes(op)
    chain_pos = {}
    for h, chains in arrays[MotifKind.DANGLING_TWO_CHAIN]:
        nodes = np.asarray([v for ch in chains for v in ch], dtype=np.int64)
        if claimed[nodes].any():
            continue
        claimed[nodes] = True
        for mo in sorted((0, 1), key=lambda m: modes[m][0]):
            _, alpha, beta = modes[mo]
            p = next_pos
            next_pos += 1
            chain_pos[p] = h
            removed[float(modes[mo][0])] += len(chains) - 1
            for k, amp in enumerate(_helmert_rows(len(chains)), start=1):
                ent = {}
                for a, (x, b) in zip(amp, chains):
                    if a != 0.0:
                        ent[x] = float(a * alpha)
                        ent[b] = float(a * beta)
                ks = sorted(ent)
                blocks.append((np.array([p]), k, np.array([ks], dtype=np.int64),
                               np.array([[ent[q] for q in ks]])))
    if not blocks:
        return None
    worst = 0.0
    for _, _, _, val in blocks:
        worst = max(worst, float(np.max(np.abs(np.einsum("ij,ij->i", val, val) - 1.0))))
    # chain modes of one hub overlap: eigenvectors of a symmetric 2x2, so
    # orthogonal; checked numerically like motifs.py:377-398
    by_hub = defaultdict(list)
    for pos, k, idx, val in blocks:
        if pos.size == 1 and int(pos[0]) in chain_pos:
            by_hub[chain_pos[int(pos[0])]].append((int(pos[0]), idx[0], val[0]))
    for vecs in by_hub.values():
        for a in range(len(vecs)):
            for b in range(a + 1, len(vecs)):
                if vecs[a][0] == vecs[b][0]:
                    continue
                _, pa, pb = np.intersect1d(vecs[a][1], vecs[b][1], return_indices=True)
                if pa.size:
                    worst = max(worst, abs(float(vecs[a][2][pa] @ vecs[b][2][pb])))
    if worst > reorth_tol:
        return None
    vpos = np.concatenate([b[0] for b in blocks])
    vk = np.concatenate([np.full(b[0].size, b[1]) for b in blocks])
    vlen = np.concatenate([np.full(b[0].size, b[2].shape[1]) for b in blocks])
    eidx = np.concatenate([b[2].reshape(-1) for b in blocks])
    evals = np.concatenate([np.ascontiguousarray(b[3]).reshape(-1) for b in blocks])
    estart = np.concatenate([[0], np.cumsum(vlen)[:-1]])
    vorder = np.lexsort((vk, vpos))
    lens_o = vlen[vorder]
    vec_ptr = np.concatenate([[0], np.cumsum(lens_o)]).astype(np.int64)
    gather = (np.repeat(estart[vorder], lens_o) +
              (np.arange(int(lens_o.sum())) - np.repeat(vec_ptr[:-1], lens_o)))
    gkey = np.arange(next_pos, dtype=np.int64)
    for p, h in chain_pos.items():
        gkey[p] = next_pos + h  # both modes of a hub: one group
    vg = gkey[vpos[vorder]]
    brk = np.ones(vg.size, dtype=bool)
    brk[1:] = vg[1:] != vg[:-1]
    group_ptr = np.append(np.flatnonzero(brk), vg.size).astype(np.int64)
    return ((group_ptr, vec_ptr, np.ascontiguousarray(eidx[gather]),
             np.ascontiguousarray(evals[gather])), dict(removed))


def _project_csr(columns, csr, ctx=None):
    cols = np.array(columns, dtype=np.float64, order="C", copy=True)
    ctx = ctx or _lib.Context.get()
    gp, vp, vi, vv = csr
    _lib.check(_lib.load().kpm_filter_probes(
        ctx.handle, cols.shape[0], cols.shape[1], _lib.ptr(cols), cols.shape[1],
        gp.shape[0] - 1, _lib.ptr(gp), _lib.ptr(vp), _lib.ptr(vi), _lib.ptr(vv)),
        "filter_probes")
    return cols


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
    fast = None
    if isinstance(instances, MotifSet) and instances.pristine() and instances.n == probes.n:
        fast = _deflation_from_arrays(instances.arrays, probes.n, reorth_tol)
    if fast is None:
        fast = _detected_deflation(list(instances), probes.n, reorth_tol)
    if fast is not None:
        csr, removed = fast
        adj = FilterAdjustment(removed=removed, total_dim=probes.n)
        if probes.device_generated:
            # seeded Rademacher block: generate, deflate and keep it in HBM --
            # the host block is only materialised if a caller reads .columns
            from .probes import DeviceBlock
            ctx = _lib.Context.get()
            blk = DeviceBlock.rademacher(ctx, probes.n, probes.seed, probes.col_offset,
                                         probes.nz)
            gp, vp, vi, vv = csr
            _lib.check(_lib.load().kpm_filter_probes(
                ctx.handle, probes.n, probes.nz, blk.ptr, blk.ld, gp.shape[0] - 1,
                _lib.ptr(gp), _lib.ptr(vp), _lib.ptr(vi), _lib.ptr(vv)), "filter_probes")
            return ProbeMatrix(probes.n, probes.nz, probes.kind, probes.seed,
                               col_offset=probes.col_offset, device_block=blk), adj
        cols = _project_csr(probes.columns, csr)
        return with_columns(probes, cols), adj
    arrays, removed = deflation_vectors(instances, probes.n, reorth_tol)
    if not arrays:
        return probes, FilterAdjustment(removed={}, total_dim=probes.n)
    cols = project_probes(probes.columns, arrays)
    return with_columns(probes, cols), FilterAdjustment(removed=removed, total_dim=probes.n)
