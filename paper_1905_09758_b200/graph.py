"""Graph storage: the host GraphCSR of the reference API plus the device CSR.

``GraphCSR`` / ``build_csr`` keep the reference's host semantics (netdos
graph.py:18-160) so a caller's graph objects, invariants and errors are
unchanged.  ``DeviceGraph`` is the B200 side: an int64 row_ptr / int32 col_idx
/ fp64 d^-1/2 CSR resident in HBM, built either from a host GraphCSR (one H2D
copy) or directly on the device from an edge list / the R-MAT generator by the
sort-based loader in csrc/kpm_graph.cu (bit-identical to _csr_from_canonical,
graph.py:69-81).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import GraphError


@dataclass(frozen=True)
class GraphCSR:
    """Symmetric CSR adjacency (graph.py:18-66 invariants): both directions
    of each undirected edge stored, columns sorted per row, self-loops stored
    once, weights > 0."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    weights: np.ndarray
    is_weighted: bool
    _degrees: np.ndarray = field(default=None, repr=False, compare=False)
    _device: object = field(default=None, repr=False, compare=False)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    @property
    def num_edges(self) -> int:
        loops = int(np.count_nonzero(self.col_idx == self._row_of_entries()))
        return (self.nnz - loops) // 2 + loops

    def _row_of_entries(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))

    def degrees(self) -> np.ndarray:
        """D_ii = sum_j a_ij (a loop weight counted once), graph.py:47-54."""
        if self._degrees is None:
            deg = np.zeros(self.n)
            np.add.at(deg, self._row_of_entries(), self.weights)
            object.__setattr__(self, "_degrees", deg)
        return self._degrees

    def neighbor_slice(self, i: int) -> slice:
        return slice(int(self.row_ptr[i]), int(self.row_ptr[i + 1]))

    def neighbors(self, i: int) -> np.ndarray:
        return self.col_idx[self.neighbor_slice(i)]

    def edge_list(self):
        """Canonical (u, v, w) triples with u <= v, sorted."""
        rows = self._row_of_entries()
        keep = rows <= self.col_idx
        return rows[keep], self.col_idx[keep], self.weights[keep]

    @property
    def unit_weights(self) -> bool:
        return bool(self.nnz == 0 or np.all(self.weights == 1.0))

    def device(self, ctx=None) -> "DeviceGraph":
        """The HBM-resident copy (created once; unit-weight CSR)."""
        if self._device is None:
            dev = DeviceGraph.from_csr(self.n, self.row_ptr, self.col_idx, ctx=ctx)
            object.__setattr__(self, "_device", dev)
        return self._device


def _csr_from_canonical(n, u, v, w, is_weighted) -> GraphCSR:
    """Symmetric CSR from deduplicated canonical pairs u <= v (graph.py:69-81
    semantics): each pair stored in both directions (a loop once), entries
    ordered by (row, col)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    off = u != v
    rows = np.concatenate([u, v[off]])
    cols = np.concatenate([v, u[off]])
    ww = np.concatenate([w, w[off]])
    order = np.argsort(rows * np.int64(max(n, 1)) + cols, kind="stable")
    rows, cols, ww = rows[order], cols[order], ww[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return GraphCSR(n=int(n), row_ptr=row_ptr, col_idx=np.ascontiguousarray(cols),
                    weights=np.ascontiguousarray(ww), is_weighted=bool(is_weighted))


def build_csr(edges, n=None, allow_self_loops=False) -> GraphCSR:
    """Assemble a GraphCSR from (u, v) or (u, v, w) tuples (graph.py:84-160
    semantics): same-direction repeats sum their weights, an edge restated in
    the opposite direction is the same undirected edge and must carry equal
    total weight, node count is 1 + max id unless ``n`` is given."""
    us, vs, ws = [], [], []
    explicit = False
    for e in edges:
        if len(e) == 3:
            a, b, wt = e
            explicit = True
        else:
            a, b = e
            wt = 1.0
        us.append(a)
        vs.append(b)
        ws.append(wt)
    return build_csr_arrays(np.asarray(us, dtype=np.int64).reshape(-1),
                            np.asarray(vs, dtype=np.int64).reshape(-1),
                            np.asarray(ws, dtype=np.float64).reshape(-1) if explicit else None,
                            n=n, allow_self_loops=allow_self_loops,
                            _orig=(us, vs, ws))


def build_csr_arrays(u, v, w=None, n=None, allow_self_loops=False, _orig=None) -> GraphCSR:
    """Vectorised build_csr over edge arrays (w None = unit, unweighted)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    explicit = w is not None
    w = np.ones(u.shape[0]) if w is None else np.asarray(w, dtype=np.float64)
    if u.size and (u.min() < 0 or v.min() < 0):
        raise GraphError("node ids must be nonnegative")
    if np.any(w <= 0):
        bad = int(np.argmax(w <= 0))
        if _orig is not None:
            raise GraphError(f"edge ({_orig[0][bad]}, {_orig[1][bad]}) has non-positive "
                             f"weight {_orig[2][bad]}")
        raise GraphError(f"edge ({u[bad]}, {v[bad]}) has non-positive weight {w[bad]}")
    if not allow_self_loops and np.any(u == v):
        node = int(u[np.argmax(u == v)])
        raise GraphError(f"self-loop at node {node} (pass allow_self_loops to accept)")
    n_min = int(max(u.max(initial=-1), v.max(initial=-1))) + 1
    if n is None:
        n = n_min
    elif n < n_min:
        raise GraphError(f"n={n} smaller than 1 + max node id ({n_min})")
    if u.size == 0:
        return GraphCSR(n=int(n), row_ptr=np.zeros(n + 1, dtype=np.int64),
                        col_idx=np.zeros(0, dtype=np.int64), weights=np.zeros(0),
                        is_weighted=False)
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    rev = (u > v).astype(np.int64)
    key = (lo * np.int64(n) + hi) * 2 + rev
    order = np.argsort(key, kind="stable")
    ks, wsort = key[order], w[order]
    uk, first = np.unique(ks, return_index=True)
    sums = np.add.reduceat(wsort, first)
    pair = uk // 2
    upair, pfirst, pcount = np.unique(pair, return_index=True, return_counts=True)
    weight = sums[pfirst].copy()
    both = np.flatnonzero(pcount == 2)
    if both.size:
        fw, bw = sums[pfirst[both]], sums[pfirst[both] + 1]
        bad = ~np.isclose(fw, bw, rtol=1e-12, atol=0.0)
        if np.any(bad):
            i = int(both[np.argmax(bad)])
            a, b = divmod(int(upair[i]), int(n))
            raise GraphError(f"edge ({a}, {b}) restated in both directions with "
                             f"conflicting weights {sums[pfirst[i]]} != {sums[pfirst[i] + 1]}")
    is_weighted = explicit and not np.all(weight == 1.0)
    return _csr_from_canonical(n, upair // n, upair % n, weight, is_weighted)


class DeviceGraph:
    """Device-resident symmetric CSR (int64 row_ptr, int32 col_idx, fp64
    d^-1/2) behind a libkpm graph handle."""

    def __init__(self, handle, ctx, explicit=False):
        self._h = handle
        self.ctx = ctx
        self.explicit = explicit
        n, nnz, mx = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().kpm_graph_info(handle, ctypes.byref(n), ctypes.byref(nnz),
                                              ctypes.byref(mx)))
        self.n, self.nnz, self.max_degree = n.value, nnz.value, mx.value

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("device graph has been freed")
        return self._h

    # ---------------------------------------------------------- builders
    @classmethod
    def from_edges(cls, n, u, v, keep_loops=False, ctx=None) -> "DeviceGraph":
        """Canonicalise + dedup + symmetric CSR on the device (K1-K3)."""
        ctx = ctx or _lib.Context.get()
        u = _as_i64(u)
        v = _as_i64(v)
        if u.shape != v.shape:
            raise ValueError("u and v differ in length")
        h = ctypes.c_void_p()
        _lib.check(_lib.load().kpm_graph_from_edges(
            ctx.handle, int(n), _lib.ptr(u), _lib.ptr(v), int(u.shape[0]),
            1 if keep_loops else 0, ctypes.byref(h)), "graph_from_edges")
        return cls(h.value, ctx)

    @classmethod
    def from_csr(cls, n, indptr, indices, values=None, shift=0.0, scale=1.0,
                 ctx=None) -> "DeviceGraph":
        """Upload an explicit CSR; values None = implicit normalized adjacency.
        int32 `indices` go to the device as they are (no widening copy); a
        device CSR is passed as addresses: indptr an int, indices a tuple
        (address, nnz, "int32" | "int64")."""
        ctx = ctx or _lib.Context.get()
        indptr = indptr if isinstance(indptr, int) else _as_i64(indptr)
        if values is not None and not isinstance(values, int):
            values = np.ascontiguousarray(values, dtype=np.float64)
        lib = _lib.load()
        if isinstance(indices, tuple):
            addr, nnz, kind = indices
            fn = lib.kpm_graph_from_csr32 if kind == "int32" else lib.kpm_graph_from_csr
        elif isinstance(indices, np.ndarray) and indices.dtype == np.int32:
            indices = np.ascontiguousarray(indices)
            addr, nnz, fn = _lib.ptr(indices), indices.shape[0], lib.kpm_graph_from_csr32
        else:
            indices = _as_i64(indices)
            addr, nnz, fn = _lib.ptr(indices), indices.shape[0], lib.kpm_graph_from_csr
        h = ctypes.c_void_p()
        _lib.check(fn(ctx.handle, int(n), _lib.ptr(indptr), addr, int(nnz), _lib.ptr(values),
                      float(shift), float(scale), ctypes.byref(h)), "graph_from_csr")
        return cls(h.value, ctx, explicit=values is not None)

    @classmethod
    def rmat(cls, scale, edge_factor=16, seed=0, a=0.57, b=0.19, c=0.19,
             ctx=None) -> "DeviceGraph":
        """R-MAT(scale, edge_factor) drawn, symmetrised, deduplicated and
        loop-free, entirely on the device (SURVEY.md §8d C3/C5 recipe)."""
        ctx = ctx or _lib.Context.get()
        ta, tab, tabc = rmat_thresholds(a, b, c)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().kpm_graph_rmat(
            ctx.handle, int(scale), int(edge_factor) << int(scale), int(seed), ta, tab, tabc,
            ctypes.byref(h)), "graph_rmat")
        return cls(h.value, ctx)

    def prepare(self, k) -> bool:
        """Build what runs of k probe columns need beside their own buffers
        (the gather-ordered twin of a large implicit graph, kpm_graph_prepare)
        before batch sizes are derived from free memory.  True when such runs
        step on the twin."""
        twin = ctypes.c_int32(0)
        _lib.check(_lib.load().kpm_graph_prepare(self.handle, int(k), ctypes.byref(twin)),
                   "graph_prepare")
        return bool(twin.value)

    def on(self, ctx) -> "DeviceGraph":
        """This graph on context `ctx`: itself, or a cached replica copied
        device to device (peer copy over NVLink for another GPU)."""
        if ctx is self.ctx:
            return self
        reps = self.__dict__.setdefault("_replicas", {})
        rep = reps.get(id(ctx))
        if rep is None:
            h = ctypes.c_void_p()
            _lib.check(_lib.load().kpm_graph_replicate(self.handle, ctx.handle,
                                                       ctypes.byref(h)), "graph_replicate")
            rep = DeviceGraph(h.value, ctx, explicit=self.explicit)
            reps[id(ctx)] = rep
        return rep

    # ---------------------------------------------------------- exports
    def export(self):
        """(row_ptr int64, col_idx int32, dinv fp64) copied to the host."""
        rp = np.empty(self.n + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int32)
        di = np.empty(self.n, dtype=np.float64)
        _lib.check(_lib.load().kpm_graph_export(self.handle, _lib.ptr(rp), _lib.ptr(ci),
                                                _lib.ptr(di)), "graph_export")
        return rp, ci, di

    def to_host(self) -> GraphCSR:
        rp, ci, _ = self.export()
        return GraphCSR(n=self.n, row_ptr=rp, col_idx=ci.astype(np.int64),
                        weights=np.ones(self.nnz), is_weighted=False)

    def degrees(self) -> np.ndarray:
        rp, _, _ = self.export()
        return np.diff(rp).astype(np.float64)

    def free(self):
        for rep in self.__dict__.pop("_replicas", {}).values():
            rep.free()
        if self._h is not None:
            _lib.load().kpm_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def rmat_thresholds(a=0.57, b=0.19, c=0.19):
    """uint32 cut points of the R-MAT quadrant probabilities."""
    two32 = 4294967296.0
    return int(a * two32), int((a + b) * two32), int((a + b + c) * two32)


def _as_i64(x):
    if hasattr(x, "data_ptr") and not isinstance(x, np.ndarray):
        return x  # torch tensor already on the device
    return np.ascontiguousarray(x, dtype=np.int64)
