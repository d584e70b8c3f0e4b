"""Row-partitioned KPM: graphs too large to replicate.

Rank q of R owns rows [lo_q, lo_{q+1}) of H (CSR rows with GLOBAL column ids)
and the matching row block of every recurrence vector.  The fused step kernel
gathers a neighbour row from whichever block owns it -- a peer GPU's memory
mapped through CUDA IPC (NVLink/NVSwitch loads; the halo exchange is the
kernel's own peer reads, overlapped tile by tile with the arithmetic) or, when
all R partitions live on one device, another block in the same HBM.  Ranks
advance in lockstep (a barrier between steps), global moments come back as raw
per-partition sums that are added in partition order and only then go through
the doubling transform, and LDOS rows are simply each partition's own rows.

``PartitionedOperator`` drives R partitions inside one process on one GPU (the
single-device form, used by the tests to check every partitioned code path
against the unpartitioned run bit for bit); ``distributed.
dos_moments_row_partitioned`` runs one partition per process.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import RecurrenceBlowupError
from .graph import DeviceGraph, rmat_thresholds
from .kpm import _BLOWUP, MODE_GLOBAL, MODE_PER_NODE, ChebMoments, Run
from .operators import ScaleMap

MAX_PARTS = 16


def balanced_bounds(row_ptr, nparts, row_cost=8):
    """Contiguous row ranges with ~equal nnz + row_cost*rows (graph-only)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = row_ptr.shape[0] - 1
    cost = row_ptr + row_cost * np.arange(n + 1, dtype=np.int64)
    targets = cost[-1] * np.arange(1, nparts, dtype=np.float64) / nparts
    cuts = np.searchsorted(cost, targets, side="left")
    return np.concatenate([[0], cuts, [n]]).astype(np.int64)


class _Part(DeviceGraph):
    """One partition's device graph (rows [row0, row0+n), global columns)."""

    def __init__(self, handle, ctx):
        super().__init__(handle, ctx)
        r0, ng = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().kpm_graph_part_info(handle, ctypes.byref(r0), ctypes.byref(ng)))
        self.row0, self.n_global = r0.value, ng.value

    def set_dinv(self, dinv_global):
        d = np.ascontiguousarray(dinv_global, dtype=np.float64)
        _lib.check(_lib.load().kpm_graph_set_dinv(self.handle, _lib.ptr(d)), "graph_set_dinv")


def part_from_csr(n_global, lo, hi, row_ptr, col_idx, values=None, shift=0.0, scale=1.0,
                  ctx=None) -> _Part:
    """Rows [lo, hi) of a global CSR as a device partition."""
    ctx = ctx or _lib.Context.get()
    rp = np.ascontiguousarray(row_ptr[lo:hi + 1] - row_ptr[lo], dtype=np.int64)
    ci = np.ascontiguousarray(col_idx[row_ptr[lo]:row_ptr[hi]], dtype=np.int64)
    vals = None if values is None else np.ascontiguousarray(
        values[row_ptr[lo]:row_ptr[hi]], dtype=np.float64)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().kpm_graph_from_csr_part(
        ctx.handle, int(n_global), int(lo), int(hi - lo), _lib.ptr(rp), _lib.ptr(ci),
        int(ci.shape[0]), _lib.ptr(vals), float(shift), float(scale), ctypes.byref(h)),
        "graph_from_csr_part")
    return _Part(h.value, ctx)


def part_rmat(scale, edge_factor, seed, lo, hi, a=0.57, b=0.19, c=0.19, ctx=None) -> _Part:
    """Rows [lo, hi) of DeviceGraph.rmat(scale, edge_factor, seed), built from
    the same draw stream on this device."""
    ctx = ctx or _lib.Context.get()
    ta, tab, tabc = rmat_thresholds(a, b, c)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().kpm_graph_rmat_part(
        ctx.handle, int(scale), int(edge_factor) << int(scale), int(seed), ta, tab, tabc,
        int(lo), int(hi), ctypes.byref(h)), "graph_rmat_part")
    return _Part(h.value, ctx)


def doubling_transform(raw, m_max):
    """Raw per-step sums -> moments (finalize_kernel's arithmetic): row 1 = S1,
    row 2 = 2 S2 - mu0; rows 2s-1 / 2s = 2 S - mu1 / 2 S - mu0 for s >= 2."""
    out = raw.copy()
    mu0, mu1 = raw[0].copy(), raw[1].copy() if m_max >= 1 else None
    for s in range(1, (m_max + 1) // 2 + 1):
        r1, r2 = 2 * s - 1, 2 * s
        if r1 <= m_max and s > 1:
            out[r1] = 2.0 * raw[r1] - mu1
        if r2 <= m_max:
            out[r2] = 2.0 * raw[r2] - mu0
    return out


class PartitionedOperator:
    """R row partitions of H = D^-1/2 A D^-1/2 on one device (or, with
    explicit values / shift / scale, any operator kind)."""

    def __init__(self, parts, bounds, shift=0.0, scale=1.0):
        self.parts = parts
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.n = int(self.bounds[-1])
        self.shift, self.scale = shift, scale
        if len(parts) > MAX_PARTS:
            raise ValueError(f"at most {MAX_PARTS} partitions")

    @property
    def scale_map(self):
        return ScaleMap(self.shift, self.scale)

    @classmethod
    def from_graph(cls, g, nparts, ctx=None):
        """Partition a host GraphCSR (unit weights) into nparts row blocks."""
        bounds = balanced_bounds(g.row_ptr, nparts)
        parts = [part_from_csr(g.n, int(bounds[q]), int(bounds[q + 1]), g.row_ptr, g.col_idx,
                               ctx=ctx) for q in range(nparts)]
        op = cls(parts, bounds)
        op._share_dinv()
        return op

    @classmethod
    def rmat(cls, scale, edge_factor, seed, nparts, ctx=None):
        n = 1 << scale
        bounds = np.linspace(0, n, nparts + 1).astype(np.int64)
        parts = [part_rmat(scale, edge_factor, seed, int(bounds[q]), int(bounds[q + 1]), ctx=ctx)
                 for q in range(nparts)]
        op = cls(parts, bounds)
        op._share_dinv()
        return op

    def _share_dinv(self):
        """All-gather d^-1/2: each partition computed its own rows' part."""
        dinv = np.concatenate([p.export()[2] for p in self.parts])
        for p in self.parts:
            p.set_dinv(dinv)

    def export(self):
        """Global (row_ptr, col_idx, dinv) assembled from the partitions."""
        rps, cis, dis = zip(*(p.export() for p in self.parts))
        off = np.cumsum([0] + [c.shape[0] for c in cis])
        rp = np.concatenate([rps[0]] + [r[1:] + o for r, o in zip(rps[1:], off[1:])])
        return rp, np.concatenate(cis), np.concatenate(dis)

    # ------------------------------------------------------------ runs
    def _runs(self, probes, mode, m_max, flags=0):
        runs = [Run(p, probes.nz, mode, m_max, flags) for p in self.parts]
        for q, (p, run) in enumerate(zip(self.parts, runs)):
            lo, hi = int(self.bounds[q]), int(self.bounds[q + 1])
            if probes.device_generated:
                run.set_probes(probes)  # device Rademacher rows [lo, hi)
            else:
                z = np.ascontiguousarray(probes.columns[lo:hi])
                run.set_probe_block(z, z.shape[1])
        blocks = []
        for run in runs:
            a, b = ctypes.c_void_p(), ctypes.c_void_p()
            _lib.check(_lib.load().kpm_run_blocks(run._h, ctypes.byref(a), ctypes.byref(b)))
            blocks.append((a.value, b.value))
        pa = (ctypes.c_void_p * len(runs))(*[x[0] for x in blocks])
        pb = (ctypes.c_void_p * len(runs))(*[x[1] for x in blocks])
        lo = np.ascontiguousarray(self.bounds, dtype=np.int64)
        for q, run in enumerate(runs):
            _lib.check(_lib.load().kpm_run_set_partition(
                run._h, len(runs), _lib.ptr(lo), q, ctypes.cast(pa, ctypes.c_void_p),
                ctypes.cast(pb, ctypes.c_void_p)), "run_set_partition")
        return runs

    @staticmethod
    def _lockstep(runs):
        total = runs[0].total_steps
        for _ in range(total):
            for run in runs:  # same stream: step k of every partition before k+1
                run.advance(1)

    def dos_contrib(self, probes, m_max, doubling=True):
        mode = _lib.MODE_DOS_DOUBLING if doubling else _lib.MODE_DOS_DIRECT
        runs = self._runs(probes, mode, m_max)
        try:
            self._lockstep(runs)
            raw = np.zeros((m_max + 1, probes.nz))
            for run in runs:  # partition order: deterministic
                part = np.empty((m_max + 1, probes.nz))
                run.result(part)
                raw += part
        finally:
            for run in runs:
                run.free()
        return doubling_transform(raw, m_max) if doubling else raw

    def dos_moments(self, probes, m_max, effective_dim=None, doubling=True) -> ChebMoments:
        contrib = self.dos_contrib(probes, m_max, doubling)
        if not np.all(np.isfinite(contrib)):
            raise RecurrenceBlowupError(_BLOWUP)
        denom = float(effective_dim) if effective_dim is not None else float(self.n)
        return ChebMoments(mode=MODE_GLOBAL, values=contrib.sum(axis=1) *
                           (probes.trace_scale / denom), scale_map=self.scale_map,
                           probe_meta=probes.meta())

    def pdos_moments(self, probes, m_max, normalized=True) -> ChebMoments:
        runs = self._runs(probes, _lib.MODE_LDOS, m_max, 0 if normalized else _lib.LDOS_RAW)
        try:
            self._lockstep(runs)
            vals = []
            for q, run in enumerate(runs):
                part = np.empty((int(self.bounds[q + 1] - self.bounds[q]), m_max + 1))
                run.result(part, probes.trace_scale)
                vals.append(part)
        finally:
            for run in runs:
                run.free()
        return ChebMoments(mode=MODE_PER_NODE, values=np.ascontiguousarray(np.concatenate(vals)),
                           scale_map=self.scale_map, probe_meta=probes.meta())

    def step_blocks(self, probes, mode, steps, m_max):
        """T_steps (global rows, host) -- for bit-exactness tests."""
        runs = self._runs(probes, mode, m_max)
        try:
            for _ in range(steps):
                for run in runs:
                    run.advance(1)
            out = []
            for run in runs:
                ptr, ld, _ = run.block()
                blk = np.empty((run.dev.n, ld))
                ctx = run.dev.ctx
                _lib.check(_lib.load().kpm_memcpy(ctx.handle, _lib.ptr(blk), ptr, blk.nbytes, 1))
                ctx.synchronize()
                out.append(blk[:, : probes.nz])
        finally:
            for run in runs:
                run.free()
        return np.concatenate(out)
