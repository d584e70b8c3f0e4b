"""Lanczos factorisations and Gauss quadrature on the B200 (SURVEY.md §8f
row 4; the reference's lanczos.py API).

Every factorisation runs in libkpm (`kpm_lanczos`): the operator's SpMV
(bit-identical to the reference's apply), the two classical Gram-Schmidt
passes against the full basis held in HBM, the residual norms and the
breakdown test -- for a whole block of start vectors at once (GQL averages
over probe columns, so all of them run in one lockstep pass).  Only the
(steps x steps) tridiagonal eigenproblems stay on the host (scipy), as in the
reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
from scipy.linalg import eigh_tridiagonal

from . import _lib
from .density import SpectralHistogram
from .errors import SpectralRangeError
from .kpm import MODE_GLOBAL, ChebMoments, chebyshev_values
from .operators import IDENTITY_MAP
from .probes import ProbeMatrix

__all__ = ["LanczosFactorization", "RitzQuadrature", "lanczos_factorize",
           "lanczos_factorize_block", "lanczos_quadrature", "gql_dos", "gql_pdos",
           "quadrature_to_cheb_moments"]

BREAKDOWN_RTOL = 1e-12


@dataclass
class LanczosFactorization:
    """Tridiagonal coefficients of H on a Krylov space (lanczos.py:27-43)."""

    alphas: np.ndarray
    betas: np.ndarray
    z_norm: float
    basis: np.ndarray | None
    exhausted: bool

    @property
    def steps(self) -> int:
        return int(self.alphas.shape[0])

    def ritz_values(self) -> np.ndarray:
        if self.steps == 1:
            return self.alphas.copy()
        return eigh_tridiagonal(self.alphas, self.betas, eigvals_only=True)


@dataclass
class RitzQuadrature:
    """Gauss rule z^T f(H) z ~= z_norm_sq * sum_i weights_i f(nodes_i)."""

    nodes: np.ndarray
    weights: np.ndarray
    z_norm_sq: float
    exhausted: bool = False


def _device_operator(op):
    """The HBM form of `op` (cached on the operator object)."""
    if hasattr(op, "device_graph"):
        return op.device_graph()
    dev = getattr(op, "_lanczos_dev", None)
    if dev is None:
        from .graph import DeviceGraph
        dev = DeviceGraph.from_csr(op.n, op.indptr, op.indices, op.data)
        try:
            op._lanczos_dev = dev
        except AttributeError:
            pass
    return dev


def _block_batch(dev, n, steps, k):
    """Columns per kpm_lanczos call: basis + residual + partial sums in HBM."""
    free, _ = _lib.Context.get().mem_info()
    per_col = 8 * n * (steps + 1) + 8 * ((n + 2047) // 2048) * (steps + 1)
    return max(1, min(k, int(0.8 * free) // max(per_col, 1)))


def lanczos_factorize_block(op, z, steps, keep_basis=False, threads=1):
    """lanczos_factorize for every column of the n x k block z; returns a
    list of LanczosFactorization (one per column)."""
    del threads
    if steps < 1:
        raise ValueError("steps must be >= 1")
    z = np.asarray(z, dtype=np.float64)
    if z.ndim == 1:
        z = z[:, None]
    n, k = z.shape
    norms = [float(np.linalg.norm(z[:, c])) for c in range(k)]
    if any(v == 0.0 for v in norms):
        raise ValueError("starting vector must be nonzero")
    dev = _device_operator(op)
    if dev.n != n:
        raise ValueError("probe dimension does not match operator")
    s = min(steps, n)
    out = []
    lib = _lib.load()
    batch = _block_batch(dev, n, s, k)
    for c0 in range(0, k, batch):
        c1 = min(k, c0 + batch)
        kb = c1 - c0
        zb = np.ascontiguousarray(z[:, c0:c1])
        zn = np.asarray(norms[c0:c1], dtype=np.float64)
        alphas = np.zeros((kb, s))
        betas = np.zeros((kb, max(s - 1, 1)))
        taken = np.zeros(kb, dtype=np.int32)
        exh = np.zeros(kb, dtype=np.int32)
        status = np.zeros(kb, dtype=np.int32)
        basis = np.empty((kb, s, n)) if keep_basis else None
        _lib.check(lib.kpm_lanczos(dev.handle, _lib.ptr(zb), kb, kb, s, _lib.ptr(zn),
                                   _lib.ptr(alphas), _lib.ptr(betas), _lib.ptr(taken),
                                   _lib.ptr(exh), _lib.ptr(status), _lib.ptr(basis)),
                   "lanczos")
        for c in range(kb):
            t = int(taken[c])
            if status[c] == 1:
                raise SpectralRangeError("NaN in Lanczos coefficients", iterations=t)
            if status[c] == 2:
                raise SpectralRangeError("NaN in Lanczos residual", iterations=t)
            out.append(LanczosFactorization(
                alphas=alphas[c, :t].copy(), betas=betas[c, :t - 1].copy(),
                z_norm=norms[c0 + c],
                basis=basis[c, :t].T.copy() if keep_basis else None,
                exhausted=bool(exh[c])))
    return out


def lanczos_factorize(op, z, steps, keep_basis=False, threads=1) -> LanczosFactorization:
    """`steps` Lanczos iterations from z with full reorthogonalisation
    (lanczos.py:46-91)."""
    z = np.asarray(z, dtype=np.float64)
    if z.ndim != 1:
        raise ValueError("z must be a vector")
    return lanczos_factorize_block(op, z, steps, keep_basis=keep_basis, threads=threads)[0]


def _quadrature(fact: LanczosFactorization) -> RitzQuadrature:
    if fact.steps == 1:
        nodes, weights = fact.alphas.copy(), np.ones(1)
    else:
        nodes, vecs = eigh_tridiagonal(fact.alphas, fact.betas)
        weights = vecs[0, :] ** 2
    return RitzQuadrature(nodes=nodes, weights=weights, z_norm_sq=fact.z_norm ** 2,
                          exhausted=fact.exhausted)


def lanczos_quadrature(op, z, steps, threads=1) -> RitzQuadrature:
    """M-step Gauss rule for the spectral measure of H weighted by z
    (lanczos.py:104-119); the truncated rule on breakdown."""
    return _quadrature(lanczos_factorize(op, z, steps, threads=threads))


def gql_dos(op, probes: ProbeMatrix, steps, bins=50, spectral_range=None,
            threads=1) -> SpectralHistogram:
    """Probe-averaged Ritz point masses binned into a density histogram
    (lanczos.py:122-141); all probe columns factorised in one device pass."""
    if op.n != probes.n:
        raise ValueError("probe dimension does not match operator")
    facts = lanczos_factorize_block(op, probes.columns, steps, threads=threads)
    quads = [_quadrature(f) for f in facts]
    nodes = np.concatenate([q.nodes for q in quads])
    weights = np.concatenate([q.weights / probes.nz for q in quads])
    if spectral_range is None:
        lo, hi = float(nodes.min()), float(nodes.max())
        pad = 1e-9 * max(hi - lo, 1.0)
        spectral_range = (lo - pad, hi + pad)
    edges = np.linspace(spectral_range[0], spectral_range[1], bins + 1)
    masses, _ = np.histogram(nodes, bins=edges, weights=weights)
    return SpectralHistogram(edges=edges, masses=masses, normalization=float(weights.sum()))


def gql_pdos(op, node, steps, threads=1) -> RitzQuadrature:
    """Quadrature for the density at one node (start vector e_node)."""
    if not 0 <= node < op.n:
        raise ValueError(f"node {node} out of range")
    e = np.zeros(op.n)
    e[node] = 1.0
    return lanczos_quadrature(op, e, steps, threads=threads)


def quadrature_to_cheb_moments(quad: RitzQuadrature, m_max, scale_map=None,
                               tol=1e-8) -> ChebMoments:
    """Chebyshev moments d_m = sum_i w_i T_m(x_i) of a Ritz rule."""
    smap = IDENTITY_MAP if scale_map is None else scale_map
    x = smap.to_scaled(quad.nodes)
    if np.any(x < -1.0 - tol) or np.any(x > 1.0 + tol):
        worst = float(x[np.argmax(np.abs(x))])
        raise ValueError(f"quadrature node {worst} outside [-1, 1] after scaling")
    values = chebyshev_values(m_max, np.clip(x, -1.0, 1.0)) @ quad.weights
    return ChebMoments(mode=MODE_GLOBAL, values=values, scale_map=smap,
                       probe_meta={"kind": "gql", "nodes": int(quad.nodes.shape[0])})
