"""Config generators and desk-scale ground truth (netdos testkit.py API).

* ``erdos_renyi`` / ``preferential_attachment`` reproduce the reference
  generators (testkit.py:149-198) draw-for-draw -- same numpy Generator calls
  in the same order -- so configs C1, C2 and C4 are the reference's graphs
  (pinned by SHA-256 digests in tests/golden/golden.json);
* ``rmat`` builds configs C3/C5 entirely on the B200 (the reference has no
  R-MAT; SURVEY.md §9.2 -- generator, dedup policy and the absence of vertex
  permutation are harness decisions recorded in DESIGN.md);
* ``motif_heavy`` builds config C4 (BA + pendant-twin pairs + 4-node stars);
* ``exact_spectrum`` & co. are the dense oracle used by the reference's tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import DeviceGraph, GraphCSR, _csr_from_canonical
from .kpm import chebyshev_values

DENSE_ORACLE_CAP = 5000


# ------------------------------------------------------------- generators
def erdos_renyi(n, p, seed=0) -> GraphCSR:
    """G(n, p): binomial edge count k, then the first k distinct values of a
    uniform stream over the n(n-1)/2 pair indices (testkit.py:149-172)."""
    if not 0.0 <= p <= 1.0:
        raise ValueError(f"p must be in [0, 1], got {p}")
    if n < 1:
        raise ValueError("n must be >= 1")
    rng = np.random.default_rng(seed)
    total = n * (n - 1) // 2
    k = int(rng.binomial(total, p)) if total else 0
    if k == 0:
        return _csr_from_canonical(n, np.zeros(0, np.int64), np.zeros(0, np.int64),
                                   np.zeros(0), False)
    chosen = np.zeros(0, dtype=np.int64)
    while chosen.size < k:
        need = k - chosen.size
        draw = rng.integers(0, total, size=need + max(16, need // 8))
        # distinct values in stream order that were not seen before
        uniq, first = np.unique(draw, return_index=True)
        fresh = ~np.isin(uniq, chosen)
        cand = uniq[fresh][np.argsort(first[fresh], kind="stable")]
        chosen = np.concatenate([chosen, cand[:need]])
    t = np.sort(chosen)
    rows = np.arange(n - 1, dtype=np.int64)
    base = rows * (2 * n - rows - 1) // 2          # first linear index of row u
    u = np.searchsorted(base, t, side="right") - 1
    v = t - base[u] + u + 1
    return _csr_from_canonical(n, u, v, np.ones(k), False)


def preferential_attachment(n, m, seed=0, native=True) -> GraphCSR:
    """Growth model (testkit.py:175-198): complete seed graph on m+1 nodes,
    then each new node picks m distinct degree-proportional targets by
    drawing uniformly from the endpoint list."""
    if m < 1 or m >= n:
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    rng = np.random.default_rng(seed)
    n_seed = m * (m + 1) // 2
    n_edges = n_seed + (n - m - 1) * m
    if native and 2 * n_edges < (1 << 32):
        # libkpm's host generator: same PCG64 stream, same draws, ~100x faster
        from . import _lib
        st = rng.bit_generator.state
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        mask = (1 << 64) - 1
        pcg = np.array([s >> 64, s & mask, inc >> 64, inc & mask, st["has_uint32"],
                        st["uinteger"]], dtype=np.uint64)
        us = np.empty(n_edges, dtype=np.int64)
        vs = np.empty(n_edges, dtype=np.int64)
        _lib.check(_lib.load().kpm_gen_preferential_attachment(
            n, m, _lib.ptr(pcg), _lib.ptr(us), _lib.ptr(vs)), "preferential_attachment")
        return _csr_from_canonical(n, us, vs, np.ones(n_edges), False)
    us = np.empty(n_edges, dtype=np.int64)
    vs = np.empty(n_edges, dtype=np.int64)
    ends = np.empty(2 * n_edges, dtype=np.int64)
    e = 0
    for a in range(m + 1):
        for b in range(a + 1, m + 1):
            us[e], vs[e] = a, b
            ends[2 * e], ends[2 * e + 1] = a, b
            e += 1
    draw = rng.integers
    for v in range(m + 1, n):
        length = 2 * e
        picked = set()
        while len(picked) < m:
            picked.add(int(ends[draw(0, length)]))
        for t in sorted(picked):
            us[e], vs[e] = t, v
            ends[2 * e], ends[2 * e + 1] = t, v
            e += 1
    return _csr_from_canonical(n, us, vs, np.ones(n_edges), False)


def rmat(scale, edge_factor=16, seed=0, a=0.57, b=0.19, c=0.19, ctx=None) -> DeviceGraph:
    """R-MAT graph generated, symmetrised, deduplicated and loop-free on the
    device (configs C3: scale 24 seed 2, C5: scale 26 seed 4)."""
    return DeviceGraph.rmat(scale, edge_factor, seed, a, b, c, ctx=ctx)


def motif_heavy_edges(n_ba=2_000_000, m=4, seed=3, twin_pairs=500_000, stars=100_000):
    """Config C4 edge list: BA(n_ba, m, seed) + `twin_pairs` pendant-twin
    pairs (two new degree-1 leaves on a uniform BA hub) + `stars` K_{1,3}
    stars (a new centre with three new leaves, the centre joined to a uniform
    BA vertex).  Attachment draws come from default_rng([seed, 0xC4]).
    Returns (n, u, v) canonical pairs."""
    g = preferential_attachment(n_ba, m, seed=seed)
    bu, bv, _ = g.edge_list()
    rng = np.random.default_rng([seed, 0xC4])
    hubs = rng.integers(0, n_ba, size=twin_pairs)
    att = rng.integers(0, n_ba, size=stars)
    leaf = n_ba + 2 * np.arange(twin_pairs, dtype=np.int64)
    pu = np.concatenate([hubs, hubs])
    pv = np.concatenate([leaf, leaf + 1])
    c = n_ba + 2 * twin_pairs + 4 * np.arange(stars, dtype=np.int64)
    su = np.concatenate([att, c, c, c])
    sv = np.concatenate([c, c + 1, c + 2, c + 3])
    u = np.concatenate([bu, pu, su]).astype(np.int64)
    v = np.concatenate([bv, pv, sv]).astype(np.int64)
    n = n_ba + 2 * twin_pairs + 4 * stars
    return n, np.minimum(u, v), np.maximum(u, v)


def motif_heavy(n_ba=2_000_000, m=4, seed=3, twin_pairs=500_000, stars=100_000) -> GraphCSR:
    n, u, v = motif_heavy_edges(n_ba, m, seed, twin_pairs, stars)
    return _csr_from_canonical(n, u, v, np.ones(u.shape[0]), False)


_MODEL_ALIASES = {
    "er": "erdos_renyi", "erdos_renyi": "erdos_renyi", "erdos-renyi": "erdos_renyi",
    "pa": "preferential_attachment", "ba": "preferential_attachment",
    "preferential_attachment": "preferential_attachment",
}


def generate_graph(model, seed=0, **params) -> GraphCSR:
    name = _MODEL_ALIASES.get(str(model).lower())
    if name is None:
        raise ValueError(f"unknown graph model {model!r}")
    return {"erdos_renyi": erdos_renyi,
            "preferential_attachment": preferential_attachment}[name](seed=seed, **params)


# --------------------------------------------------------- dense oracle
@dataclass
class ExactSpectrum:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray | None = None


def dense_matrix(op) -> np.ndarray:
    """Materialise an operator by applying it to the identity."""
    return np.asarray(op.apply(np.eye(op.n)))


def exact_spectrum(op, want_vectors=False, cap=DENSE_ORACLE_CAP) -> ExactSpectrum:
    from scipy.linalg import eigh

    if op.n > cap:
        raise ValueError(f"oracle capped at {cap} nodes (got {op.n}); "
                         "it exists for validation, not production")
    h = dense_matrix(op)
    if want_vectors:
        vals, vecs = eigh(h)
        return ExactSpectrum(eigenvalues=vals, eigenvectors=vecs)
    return ExactSpectrum(eigenvalues=eigh(h, eigvals_only=True))


def oracle_histogram(eigenvalues, edges, snap=1e-9) -> np.ndarray:
    ev = np.asarray(eigenvalues, dtype=np.float64).copy()
    edges = np.asarray(edges, dtype=np.float64)
    if snap:
        pos = np.searchsorted(edges, ev)
        for cand in (np.clip(pos - 1, 0, len(edges) - 1), np.clip(pos, 0, len(edges) - 1)):
            near = np.abs(ev - edges[cand]) <= snap
            ev[near] = edges[cand[near]]
    masses, _ = np.histogram(ev, bins=edges)
    return masses / float(len(ev))


def oracle_moments(eigenvalues_scaled, m_max) -> np.ndarray:
    return chebyshev_values(m_max, eigenvalues_scaled).mean(axis=1)
