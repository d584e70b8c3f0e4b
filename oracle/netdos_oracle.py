"""CPU oracle for the KPM hot path -- TEST INFRASTRUCTURE ONLY.

Restates the reference (netdos 0.1.0, /root/reference/pkg/src/netdos) algorithm
for the Chebyshev-moment path in numpy plus the plain-C helpers of
``oracle/kpm_oracle.c``.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker or the timed CPU baseline: the shipped package
``paper_1905_09758_b200`` never imports it and has no CPU fallback.

Parity of this restatement is pinned by ``tests/test_oracle.py`` against
fixtures written by the reference itself (``tests/golden/make_golden.py``).

Two SpMM engines are available to the restated recurrence:
* ``"ref"``: the reference's OWN compiled kernel, ``_spmv.pyx`` -> ``_spmv.c``
  built unchanged by ``oracle/build_ref.sh`` into ``oracle/_ref/`` (present on
  the GPU box because built files travel with the snapshot);
* ``"c"``: ``orc_csr_matvec`` in ``kpm_oracle.c`` (same arithmetic).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)

_lib = None
_ref = None


def _ptr(a, t):
    return a.ctypes.data_as(t)


def build():
    """Compile libkpm_oracle.so (and oracle/_ref when the reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "libkpm_oracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.orc_csr_from_edges.restype = ctypes.c_int64
        L.orc_csr_from_edges.argtypes = [ctypes.c_int64, _I64P, _I64P, ctypes.c_int64,
                                         ctypes.c_int, _I64P, _I64P]
        L.orc_dinv.restype = None
        L.orc_dinv.argtypes = [ctypes.c_int64, _I64P, _F64P]
        L.orc_normadj_values.restype = None
        L.orc_normadj_values.argtypes = [ctypes.c_int64, _I64P, _I64P, _F64P, _F64P]
        L.orc_csr_matvec.restype = None
        L.orc_csr_matvec.argtypes = [ctypes.c_int64, _I64P, _I64P, _F64P, _F64P,
                                     ctypes.c_int64, _F64P, ctypes.c_int]
        for name in ("orc_dos_contrib", "orc_ldos_num"):
            f = getattr(L, name)
            f.restype = None
            f.argtypes = [ctypes.c_int64, _I64P, _I64P, _F64P, ctypes.c_double,
                          ctypes.c_double, _F64P, ctypes.c_int64, ctypes.c_int, _F64P,
                          ctypes.c_int]
        L.orc_recurrence_block.restype = None
        L.orc_recurrence_block.argtypes = [ctypes.c_int64, _I64P, _I64P, _F64P,
                                           ctypes.c_double, ctypes.c_double, _F64P,
                                           ctypes.c_int64, ctypes.c_int, _F64P, ctypes.c_int]
        L.orc_rmat_edges.restype = None
        L.orc_rmat_edges.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                     ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int64,
                                     ctypes.c_int64, _I64P, _I64P, ctypes.c_int]
        _lib = L
    return _lib


def ref_spmv():
    """The reference's compiled Cython kernel module (oracle/_ref), or None."""
    global _ref
    if _ref is None:
        cands = glob.glob(os.path.join(HERE, "_ref", "_spmv*.so"))
        if not cands:
            return None
        name = "netdos._kernels._spmv"
        spec = importlib.util.spec_from_file_location(name, cands[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules.setdefault(name, mod)
        _ref = mod
    return _ref


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------- graph / CSR
def csr_from_canonical(n, u, v):
    """graph.py:69-81 _csr_from_canonical (unit weights), numpy restatement."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    loops = u == v
    ru = np.concatenate([u, v[~loops]])
    cv = np.concatenate([v, u[~loops]])
    order = np.lexsort((cv, ru))
    ru, cv = ru[order], cv[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, ru + 1, 1)
    np.cumsum(row_ptr, out=row_ptr)
    return row_ptr, cv.astype(np.int64)


def canonical_pairs(u, v, drop_loops=True):
    """(min, max), drop u == v, np.unique on u*n+v: the harness dedup step
    applied to raw generator output before _csr_from_canonical."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    a, b = np.minimum(u, v), np.maximum(u, v)
    if drop_loops:
        keep = a != b
        a, b = a[keep], b[keep]
    key = np.unique((a << np.int64(32)) | b)
    return key >> np.int64(32), key & np.int64(0xFFFFFFFF)


def csr_from_edges(n, u, v, keep_loops=False):
    """C restatement: canonicalise + dedup + _csr_from_canonical in O(nnz)."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    row_ptr = np.empty(n + 1, dtype=np.int64)
    col = np.empty(max(1, 2 * u.shape[0]), dtype=np.int64)
    nnz = lib().orc_csr_from_edges(n, _ptr(u, _I64P), _ptr(v, _I64P), u.shape[0],
                                   1 if keep_loops else 0, _ptr(row_ptr, _I64P),
                                   _ptr(col, _I64P))
    if nnz < 0:
        raise ValueError("node id out of range")
    return row_ptr, col[:nnz].copy()


def degrees(row_ptr):
    """graph.py:47-54 for unit weights."""
    return np.diff(row_ptr).astype(np.float64)


def dinv_of(row_ptr):
    """operators.py:108-109."""
    deg = degrees(row_ptr)
    with np.errstate(divide="ignore"):
        return np.where(deg > 0, 1.0 / np.sqrt(np.maximum(deg, 1e-300)), 0.0)


def normadj_values(row_ptr, col_idx, dinv=None):
    """operators.py:110 norm_w = w * dinv[rows] * dinv[cols] (w = 1)."""
    if dinv is None:
        dinv = dinv_of(row_ptr)
    rows = np.repeat(np.arange(row_ptr.shape[0] - 1, dtype=np.int64), np.diff(row_ptr))
    return (1.0 * dinv[rows]) * dinv[col_idx]


def normadj_values_c(row_ptr, col_idx, dinv):
    """Same values as normadj_values (operators.py:110, (1.0*dinv[r])*dinv[c])
    from the C restatement on all host threads, without numpy's row-index
    temporaries (C5: 2.1e9 nonzeros)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    di = np.ascontiguousarray(dinv, dtype=np.float64)
    out = np.empty(ci.shape[0])
    lib().orc_normadj_values(rp.shape[0] - 1, _ptr(rp, _I64P), _ptr(ci, _I64P), _ptr(di, _F64P),
                             _ptr(out, _F64P))
    return out


# --------------------------------------------------------------------- SpMM
def csr_matvec(indptr, indices, data, x, threads=1, engine="c"):
    """_kernels/__init__.py:33-46 csr_matvec with a chosen engine."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    one_d = x.ndim == 1
    x2 = x[:, None] if one_d else x
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    data = np.ascontiguousarray(data, dtype=np.float64)
    n = indptr.shape[0] - 1
    out = np.empty((n, x2.shape[1]))
    if engine == "ref":
        mod = ref_spmv()
        if mod is None:
            raise RuntimeError("oracle/_ref not built")
        mod.csr_matvec(indptr, indices, data, np.ascontiguousarray(x2), out, int(threads))
    else:
        lib().orc_csr_matvec(n, _ptr(indptr, _I64P), _ptr(indices, _I64P),
                             _ptr(data, _F64P), _ptr(np.ascontiguousarray(x2), _F64P),
                             x2.shape[1], _ptr(out, _F64P), int(threads))
    return out[:, 0] if one_d else out


class CSROp:
    """Duck-typed stand-in for operators.SymmetricCSROperator wrapped by
    ScaledOperator (operators.py:50-65, 124-148)."""

    def __init__(self, indptr, indices, data, shift=0.0, scale=1.0, engine="c"):
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        self.n = self.indptr.shape[0] - 1
        self.shift = float(shift)
        self.scale = float(scale)
        self.engine = engine

    def apply(self, x, out=None, threads=1):
        y = csr_matvec(self.indptr, self.indices, self.data, x, threads, self.engine)
        if out is not None:
            out[...] = y
            y = out
        if self.shift != 0.0:
            y -= self.shift * x
        if self.scale != 1.0:
            y /= self.scale
        return y


def recurrence(sop, z, m_max, collect, threads=1):
    """kpm.py:73-89 _recurrence (same numpy calls, same buffer rotation)."""
    t_prev = np.array(z, dtype=np.float64, order="C", copy=True)
    collect(0, t_prev)
    if m_max == 0:
        return
    t_cur = sop.apply(t_prev, threads=threads)
    collect(1, t_cur)
    scratch = np.empty_like(t_cur)
    with np.errstate(over="ignore", invalid="ignore"):
        for m in range(2, m_max + 1):
            t_next = sop.apply(t_cur, out=scratch, threads=threads)
            t_next *= 2.0
            t_next -= t_prev
            collect(m, t_next)
            t_prev, t_cur, scratch = t_cur, t_next, t_prev


def dos_contrib(sop, z, m_max, threads=1):
    """kpm.py:104-108: the per-probe contribution matrix (m_max+1, nz)."""
    contrib = np.empty((m_max + 1, z.shape[1]))

    def collect(m, t_m):
        contrib[m] = np.einsum("ij,ij->j", z, t_m)

    recurrence(sop, z, m_max, collect, threads)
    return contrib


def dos_values(contrib, trace_scale, denom):
    """kpm.py:111-115."""
    if not np.all(np.isfinite(contrib)):
        raise FloatingPointError("Chebyshev recurrence overflowed")
    return contrib.sum(axis=1) * (trace_scale / denom)


def ldos_num(sop, z, m_max, threads=1):
    """kpm.py:133-136: num (m_max+1, n)."""
    num = np.empty((m_max + 1, sop.n))

    def collect(m, t_m):
        num[m] = np.einsum("ij,ij->i", z, t_m)

    recurrence(sop, z, m_max, collect, threads)
    return num


def pdos_values(num, z, normalized=True, trace_scale=None):
    """kpm.py:143-151."""
    if normalized:
        den = np.einsum("ij,ij->i", z, z)
        return np.ascontiguousarray((num / den).T)
    return np.ascontiguousarray((num * trace_scale).T)


def recurrence_block(sop, z, steps, threads=1):
    """T_steps(H) z exactly as kpm.py:76-89 produces it."""
    box = {}

    def collect(m, t_m):
        if m == steps:
            box["t"] = t_m.copy()

    recurrence(sop, z, steps, collect, threads)
    return box["t"]


def c_dos_contrib(indptr, indices, data, z, m_max, shift=0.0, scale=1.0, threads=1):
    """Same as dos_contrib through the plain-C restatement."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    n, k = z.shape
    out = np.empty((m_max + 1, k))
    lib().orc_dos_contrib(n, _ptr(indptr, _I64P), _ptr(indices, _I64P), _ptr(data, _F64P),
                          shift, scale, _ptr(z, _F64P), k, m_max, _ptr(out, _F64P),
                          int(threads))
    return out


def c_ldos_num(indptr, indices, data, z, m_max, shift=0.0, scale=1.0, threads=1):
    z = np.ascontiguousarray(z, dtype=np.float64)
    n, k = z.shape
    out = np.empty((m_max + 1, n))
    lib().orc_ldos_num(n, _ptr(indptr, _I64P), _ptr(indices, _I64P), _ptr(data, _F64P),
                       shift, scale, _ptr(z, _F64P), k, m_max, _ptr(out, _F64P),
                       int(threads))
    return out


def c_recurrence_block(indptr, indices, data, z, steps, shift=0.0, scale=1.0, threads=1):
    z = np.ascontiguousarray(z, dtype=np.float64)
    n, k = z.shape
    out = np.empty((n, k))
    lib().orc_recurrence_block(n, _ptr(indptr, _I64P), _ptr(indices, _I64P),
                               _ptr(data, _F64P), shift, scale, _ptr(z, _F64P), k,
                               steps, _ptr(out, _F64P), int(threads))
    return out


# ------------------------------------------------------------------- probes
def make_probes(n, nz, kind="rademacher", seed=0):
    """probes.py:52-91 make_probes (columns only)."""
    if nz < 1:
        raise ValueError("nz must be >= 1")

    def streams(count):
        return [np.random.Generator(np.random.Philox(ss))
                for ss in np.random.SeedSequence(int(seed)).spawn(count)]

    if kind == "standard-basis":
        if nz > n:
            raise ValueError(f"standard-basis probes need nz <= n (got {nz} > {n})")
        cols = np.zeros((n, nz))
        cols[np.arange(nz), np.arange(nz)] = 1.0
    elif kind == "hadamard":
        st = streams(nz + 1)
        flips = 1.0 - 2.0 * st[nz].integers(0, 2, size=n).astype(np.float64)
        size = 1 << max(1, int(np.ceil(np.log2(max(n, 2)))))
        if nz > size:
            raise ValueError(f"hadamard probes support at most {size} columns for n={n}")
        i = np.arange(n, dtype=np.uint64)[:, None]
        j = np.arange(nz, dtype=np.uint64)[None, :]
        parity = np.bitwise_count(i & j) & np.uint64(1)
        cols = flips[:, None] * (1.0 - 2.0 * parity.astype(np.float64))
    else:
        st = streams(nz)
        cols = np.empty((n, nz))
        for j, rng in enumerate(st):
            if kind == "gaussian":
                cols[:, j] = rng.standard_normal(n)
            else:
                cols[:, j] = 1.0 - 2.0 * rng.integers(0, 2, size=n).astype(np.float64)
    return np.ascontiguousarray(cols)


def rademacher_column(n, seed, j):
    """Column j alone via SeedSequence(seed, spawn_key=(j,))."""
    ss = np.random.SeedSequence(int(seed), spawn_key=(int(j),))
    rng = np.random.Generator(np.random.Philox(ss))
    return 1.0 - 2.0 * rng.integers(0, 2, size=n).astype(np.float64)


# ------------------------------------------------------------ density side
def jackson_coefficients(m_max):
    """kpm.py:48-58."""
    big_m = m_max + 1
    m = np.arange(big_m, dtype=np.float64)
    theta = np.pi * m / big_m
    out = ((big_m - m) * np.cos(theta) + np.sin(theta) / np.tan(np.pi / big_m)) / big_m
    out[0] = 1.0
    return np.maximum(out, 0.0)


def cheb_bin_masses(m_max, scaled_edges):
    """density.py:51-60."""
    theta = np.arccos(np.clip(scaled_edges, -1.0, 1.0))
    out = np.empty((m_max + 1, len(scaled_edges) - 1))
    out[0] = (theta[:-1] - theta[1:]) / np.pi
    if m_max >= 1:
        m = np.arange(1, m_max + 1, dtype=np.float64)[:, None]
        s = np.sin(m * theta[None, :])
        out[1:] = (2.0 / np.pi) * (s[:, :-1] - s[:, 1:]) / m
    return out


def histogram_masses(values, bins=50, damping=True, shift=0.0, scale=1.0,
                     removed=None, total_dim=None):
    """density.py:63-100 for a global moment vector (edges default)."""
    values = np.asarray(values, dtype=np.float64)
    m_max = values.shape[-1] - 1
    edges = shift + scale * np.linspace(-1.0, 1.0, bins + 1)
    table = cheb_bin_masses(m_max, (edges - shift) / scale)
    coef = values.copy()
    if damping:
        coef = coef * jackson_coefficients(m_max)
    masses = coef @ table
    if removed:
        r = int(sum(removed.values()))
        masses = masses * ((total_dim - r) / total_dim)
        for lam, count in sorted(removed.items()):
            i = int(np.searchsorted(edges, lam, side="right")) - 1
            masses[min(max(i, 0), len(edges) - 2)] += count / total_dim
    return edges, masses


# ------------------------------------------------------------------ Lanczos
def lanczos_factorize(apply, z, steps):
    """lanczos.py:46-91: Lanczos from z with two classical Gram-Schmidt passes
    against the whole basis; stops on a residual below 1e-12 * hnorm.
    `apply(x)` is the operator's matvec.  Returns (alphas, betas, exhausted,
    basis)."""
    z = np.asarray(z, dtype=np.float64)
    z_norm = float(np.linalg.norm(z))
    n = z.shape[0]
    steps = min(steps, n)
    basis = np.empty((n, steps))
    basis[:, 0] = z / z_norm
    alphas, betas = np.empty(steps), np.empty(max(steps - 1, 0))
    exhausted, hnorm, k = False, 0.0, 0
    for j in range(steps):
        q = basis[:, j]
        w = apply(q)
        alphas[j] = float(q @ w)
        hnorm = max(hnorm, abs(alphas[j]) + (betas[j - 1] if j > 0 else 0.0))
        k = j + 1
        if j == steps - 1:
            break
        qb = basis[:, : j + 1]
        for _ in range(2):
            w -= qb @ (qb.T @ w)
        beta = float(np.linalg.norm(w))
        if beta <= 1e-12 * max(hnorm, 1e-300):
            exhausted = True
            break
        betas[j] = beta
        hnorm = max(hnorm, beta)
        basis[:, j + 1] = w / beta
    return alphas[:k].copy(), betas[: k - 1].copy(), exhausted, basis[:, :k].copy()


def ritz_rule(alphas, betas):
    """lanczos.py:104-119: Ritz nodes and first-component weights."""
    from scipy.linalg import eigh_tridiagonal
    if alphas.shape[0] == 1:
        return alphas.copy(), np.ones(1)
    nodes, vecs = eigh_tridiagonal(alphas, betas)
    return nodes, vecs[0, :] ** 2


# ---------------------------------------------------------- motif filtering
def project_out(columns, vectors):
    """motifs.py:400-403: for each sparse (idx, val) in order,
    coeff = val @ cols[idx]; cols[idx] -= outer(val, coeff)."""
    cols = np.array(columns, dtype=np.float64, copy=True)
    for idx, val in vectors:
        coeff = val @ cols[idx]
        cols[idx] -= np.outer(val, coeff)
    return cols


# ------------------------------------------------------------------- R-MAT
def rmat_thresholds(a=0.57, b=0.19, c=0.19):
    """uint32 cut points of the quadrant probabilities (harness decision)."""
    two32 = 4294967296.0
    ta = int(a * two32)
    tab = int((a + b) * two32)
    tabc = int((a + b + c) * two32)
    return ta, tab, tabc


def rmat_edges(scale, n_edges, seed, a=0.57, b=0.19, c=0.19, e0=0, count=None,
               threads=None):
    """Raw R-MAT draws [e0, e0+count) from the counter-based generator."""
    if count is None:
        count = n_edges - e0
    u = np.empty(count, dtype=np.int64)
    v = np.empty(count, dtype=np.int64)
    ta, tab, tabc = rmat_thresholds(a, b, c)
    lib().orc_rmat_edges(int(scale), int(seed), ta, tab, tabc, int(e0), int(count),
                         _ptr(u, _I64P), _ptr(v, _I64P), int(threads or cpu_threads()))
    return u, v
