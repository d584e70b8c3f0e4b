"""Probe blocks (netdos probes.py API) with device-side Rademacher generation.

Column j of a RADEMACHER block is ``1 - 2*Philox(SeedSequence(seed).spawn(nz)[j])
.integers(0, 2, n)`` (probes.py:52-54, 86-89).  The host derives each column's
128-bit Philox key from numpy's SeedSequence ("seeded on the host"); the B200
regenerates the block from those keys bit-identically (csrc rademacher_kernel),
so a 17 GB probe block (config C3) never crosses PCIe and never occupies host
RAM.  ``ProbeMatrix.columns`` still materialises the numpy block on demand, so
the reference's host semantics are unchanged.
"""

from __future__ import annotations

from enum import Enum

import numpy as np


class ProbeKind(str, Enum):
    GAUSSIAN = "gaussian"
    RADEMACHER = "rademacher"
    HADAMARD = "hadamard"
    STANDARD_BASIS = "standard-basis"


def _streams(seed, count, col0=0):
    """Generators of columns col0..col0+count-1: SeedSequence(seed).spawn(nz)[j]
    is SeedSequence(seed, spawn_key=(j,)), so any column range is reproducible
    on its own (column stability, probes.py:1-6)."""
    return [np.random.Generator(np.random.Philox(
        np.random.SeedSequence(int(seed), spawn_key=(col0 + j,)))) for j in range(count)]


def philox_keys(seed, nz, col0=0, col1=None) -> np.ndarray:
    """uint64[2*(col1-col0)]: the Philox4x64 key of each probe column
    (SeedSequence(seed).spawn(nz)[j], column-stable)."""
    col1 = nz if col1 is None else col1
    keys = np.empty(2 * (col1 - col0), dtype=np.uint64)
    for t, j in enumerate(range(col0, col1)):
        ss = np.random.SeedSequence(int(seed), spawn_key=(j,))
        keys[2 * t: 2 * t + 2] = np.random.Philox(ss).state["state"]["key"]
    return keys


def _sylvester_columns(n, nz):
    size = 1 << max(1, int(np.ceil(np.log2(max(n, 2)))))
    if nz > size:
        raise ValueError(f"hadamard probes support at most {size} columns for n={n}")
    i = np.arange(n, dtype=np.uint64)[:, None]
    j = np.arange(nz, dtype=np.uint64)[None, :]
    parity = np.bitwise_count(i & j) & np.uint64(1)
    return 1.0 - 2.0 * parity.astype(np.float64)


def _host_columns(n, nz, kind, seed, col0=0):
    if kind is ProbeKind.STANDARD_BASIS:
        cols = np.zeros((n, nz))
        cols[np.arange(nz), np.arange(nz)] = 1.0
        return cols
    if kind is ProbeKind.HADAMARD:
        st = _streams(seed, nz + 1)
        flips = 1.0 - 2.0 * st[nz].integers(0, 2, size=n).astype(np.float64)
        return flips[:, None] * _sylvester_columns(n, nz)
    cols = np.empty((n, nz))
    for j, rng in enumerate(_streams(seed, nz, col0)):
        if kind is ProbeKind.GAUSSIAN:
            cols[:, j] = rng.standard_normal(n)
        else:
            cols[:, j] = 1.0 - 2.0 * rng.integers(0, 2, size=n).astype(np.float64)
    return np.ascontiguousarray(cols)


class ProbeMatrix:
    """n x nz probe block plus its generating metadata (probes.py:23-49).

    ``columns`` is the C-contiguous numpy block; for seeded RADEMACHER probes it
    is generated lazily (``device_generated`` is then True until materialised
    or replaced), letting the recurrence generate the block in HBM instead."""

    def __init__(self, n, nz, kind, seed, columns=None, col_offset=0, device_block=None):
        self.n = int(n)
        self.nz = int(nz)
        self.kind = ProbeKind(kind)
        self.seed = int(seed)
        self.col_offset = int(col_offset)  # first column index in the seeded family
        self._columns = None if columns is None else np.ascontiguousarray(columns)
        self.device_block = device_block  # HBM-resident columns (e.g. filtered)

    @property
    def columns(self) -> np.ndarray:
        if self._columns is None:
            if self.device_block is not None:
                self._columns = self.device_block.to_host()
            else:
                self._columns = _host_columns(self.n, self.nz, self.kind, self.seed,
                                              self.col_offset)
        return self._columns

    @property
    def device_generated(self) -> bool:
        """True while the block is still the pristine seeded Rademacher block
        (the device regenerates it from philox_keys instead of uploading)."""
        return (self._columns is None and self.device_block is None
                and self.kind is ProbeKind.RADEMACHER)

    @property
    def deterministic(self) -> bool:
        return self.kind is ProbeKind.STANDARD_BASIS

    @property
    def trace_scale(self) -> float:
        return 1.0 if self.deterministic else 1.0 / self.nz

    def meta(self) -> dict:
        return {"kind": self.kind.value, "seed": self.seed, "nz": self.nz,
                "exact": bool(self.deterministic and self.nz == self.n)}

    def keys(self) -> np.ndarray:
        if self.kind is not ProbeKind.RADEMACHER:
            raise ValueError("Philox keys exist for rademacher probes only")
        o = self.col_offset
        return philox_keys(self.seed, o + self.nz, o, o + self.nz)

    def column_slice(self, col0, col1) -> "ProbeMatrix":
        """Columns [col0, col1) as their own block (probe sharding / batching);
        a seeded Rademacher slice stays lazy and column-stable."""
        if self.device_generated:
            return ProbeMatrix(self.n, col1 - col0, self.kind, self.seed,
                               col_offset=self.col_offset + col0)
        if self._columns is None and self.device_block is not None:
            return ProbeMatrix(self.n, col1 - col0, self.kind, self.seed,
                               col_offset=self.col_offset + col0,
                               device_block=self.device_block.column_view(col0, col1))
        return ProbeMatrix(self.n, col1 - col0, self.kind, self.seed,
                           columns=np.ascontiguousarray(self.columns[:, col0:col1]),
                           col_offset=self.col_offset + col0)

    def __repr__(self):
        return (f"ProbeMatrix(n={self.n}, nz={self.nz}, kind={self.kind.value}, "
                f"seed={self.seed}, lazy={self._columns is None})")


class DeviceBlock:
    """An n x k fp64 probe block resident in HBM (row stride ld), owned by
    libkpm's allocator; column views share the allocation."""

    def __init__(self, ctx, n, k, ld=None, _base=None, _ptr=None):
        import ctypes

        from . import _lib
        self.ctx, self.n, self.k = ctx, int(n), int(k)
        self.ld = int(ld if ld is not None else k)
        self._base = _base
        if _ptr is None:
            p = ctypes.c_void_p()
            _lib.check(_lib.load().kpm_device_alloc(ctx.handle, 8 * max(self.n * self.ld, 1),
                                                    ctypes.byref(p)), "device_alloc")
            self.ptr, self._owner = p.value, True
        else:
            self.ptr, self._owner = _ptr, False

    @classmethod
    def rademacher(cls, ctx, n, seed, col0, ncols):
        """Seeded Rademacher columns generated on the device (bit-identical
        to make_probes)."""
        from . import _lib
        blk = cls(ctx, n, ncols)
        keys = philox_keys(seed, col0 + ncols, col0, col0 + ncols)
        _lib.check(_lib.load().kpm_probes_rademacher(ctx.handle, n, ncols, _lib.ptr(keys),
                                                     blk.ptr, blk.ld, 0), "probes_rademacher")
        return blk

    def column_view(self, c0, c1):
        return DeviceBlock(self.ctx, self.n, c1 - c0, self.ld, _base=self,
                           _ptr=self.ptr + 8 * c0)

    def to_host(self) -> np.ndarray:
        from . import _lib
        out = np.empty((self.n, self.ld))
        _lib.check(_lib.load().kpm_memcpy(self.ctx.handle, _lib.ptr(out), self.ptr,
                                          out.nbytes, 1), "memcpy")
        self.ctx.synchronize()
        return np.ascontiguousarray(out[:, : self.k])

    def __del__(self):
        try:
            if self._owner and self.ptr:
                from . import _lib
                _lib.load().kpm_device_free(self.ctx.handle, self.ptr)
        except Exception:
            pass


def make_probes(n, nz, kind=ProbeKind.RADEMACHER, seed=0) -> ProbeMatrix:
    """Deterministic function of (n, nz, kind, seed) (probes.py:68-91)."""
    kind = ProbeKind(kind)
    if nz < 1:
        raise ValueError("nz must be >= 1")
    if kind is ProbeKind.STANDARD_BASIS and nz > n:
        raise ValueError(f"standard-basis probes need nz <= n (got {nz} > {n})")
    if kind is ProbeKind.HADAMARD:
        size = 1 << max(1, int(np.ceil(np.log2(max(n, 2)))))
        if nz > size:
            raise ValueError(f"hadamard probes support at most {size} columns for n={n}")
    p = ProbeMatrix(n, nz, kind, seed)
    if kind is not ProbeKind.RADEMACHER:
        p.columns  # noqa: B018 -- eager, as the reference
    return p


def with_columns(probes: ProbeMatrix, columns: np.ndarray) -> ProbeMatrix:
    """Copy of ``probes`` carrying replacement columns (probes.py:94-96)."""
    return ProbeMatrix(probes.n, probes.nz, probes.kind, probes.seed,
                       columns=np.ascontiguousarray(columns))


def estimate_trace(op, probes: ProbeMatrix, threads=1) -> float:
    """Hutchinson trace estimate (probes.py:99-107)."""
    z = probes.columns
    if op.n != probes.n:
        raise ValueError("probe dimension does not match operator")
    hz = op.apply(z, threads=threads)
    return float(np.einsum("ij,ij->", z, hz) * probes.trace_scale)


def estimate_diagonal(op, probes: ProbeMatrix, normalized=True, threads=1):
    """Stochastic diagonal estimate (probes.py:110-126)."""
    z = probes.columns
    if op.n != probes.n:
        raise ValueError("probe dimension does not match operator")
    hz = op.apply(z, threads=threads)
    num = np.einsum("ij,ij->i", z, hz)
    if not normalized:
        return num * probes.trace_scale
    den = np.einsum("ij,ij->i", z, z)
    if np.any(den == 0.0):
        k = int(np.argmax(den == 0.0))
        raise ValueError(f"zero probe mass at coordinate {k}; diagonal entry unrecoverable")
    return num / den
