"""Chebyshev moments on the B200 (drop-in for netdos kpm.py).

``dos_moments`` / ``pdos_moments`` keep the reference signatures, return types
and errors (kpm.py:92-152); the recurrence itself runs in libkpm's fused
sm_100a step kernel (csrc/kpm_step.cu), one launch per step, with the probe
block resident in HBM.  Only the per-probe contribution matrix (global) or the
(n, M+1) per-node result (LDOS) comes back to the host, which finishes exactly
as the reference does (``contrib.sum(axis=1) * trace_scale / denom``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import RecurrenceBlowupError
from .operators import ScaleMap
from .probes import ProbeMatrix

MODE_GLOBAL = "global"
MODE_PER_NODE = "per_node"

_BLOWUP = ("Chebyshev recurrence overflowed; re-estimate the spectral range "
           "with a larger margin")


@dataclass
class ChebMoments:
    """Moment sequences plus the scale map needed to interpret them
    (kpm.py:24-45): values (m_max+1,) global or (n, m_max+1) per node."""

    mode: str
    values: np.ndarray
    scale_map: ScaleMap
    probe_meta: dict

    @property
    def m_max(self) -> int:
        return int(self.values.shape[-1] - 1)

    @property
    def global_values(self) -> np.ndarray:
        if self.mode == MODE_GLOBAL:
            return self.values
        return self.values.mean(axis=0)


def jackson_coefficients(m_max: int) -> np.ndarray:
    """Jackson damping J_0..J_M (kpm.py:48-58)."""
    if m_max < 0:
        raise ValueError("m_max must be >= 0")
    big = m_max + 1
    m = np.arange(big, dtype=np.float64)
    theta = np.pi * m / big
    out = ((big - m) * np.cos(theta) + np.sin(theta) / np.tan(np.pi / big)) / big
    out[0] = 1.0
    return np.maximum(out, 0.0)


def chebyshev_values(m_max: int, x) -> np.ndarray:
    """T[m, i] = T_m(x_i) by the scalar three-term recurrence (kpm.py:61-70)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    out = np.empty((m_max + 1, x.shape[0]))
    out[0] = 1.0
    if m_max >= 1:
        out[1] = x
    for m in range(2, m_max + 1):
        out[m] = 2.0 * x * out[m - 1] - out[m - 2]
    return out


# ---------------------------------------------------------------- device run
def _device_graph(sop):
    if hasattr(sop, "device_graph"):
        return sop.device_graph()
    # a foreign ScaledOperator (e.g. the reference's): explicit CSR values
    from .graph import DeviceGraph
    base = sop.base
    return DeviceGraph.from_csr(base.n, base.indptr, base.indices, base.data,
                                getattr(sop, "shift", 0.0), getattr(sop, "scale", 1.0))


class Run:
    """One probe batch through the fused recurrence (kpm_run_* C-ABI)."""

    def __init__(self, dev, k, mode, m_max, flags=0):
        self.dev = dev
        self.k = int(k)
        self.mode = mode
        self.m_max = int(m_max)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().kpm_run_create(dev.handle, self.k, mode, self.m_max, flags,
                                              ctypes.byref(h)), "run_create")
        self._h = h.value
        self.total_steps = _lib.load().kpm_run_total_steps(self._h)

    def set_probes(self, probes: ProbeMatrix):
        """Upload an explicit block, or regenerate seeded Rademacher columns
        on the device from their Philox keys."""
        if probes.device_generated:
            keys = probes.keys()
            _lib.check(_lib.load().kpm_run_set_rademacher(self._h, _lib.ptr(keys)),
                       "run_set_rademacher")
        elif probes._columns is None and probes.device_block is not None:
            blk = probes.device_block  # HBM-resident (e.g. motif-filtered): D2D
            _lib.check(_lib.load().kpm_run_set_probes(self._h, blk.ptr, blk.ld),
                       "run_set_probes")
        else:
            z = np.ascontiguousarray(probes.columns, dtype=np.float64)
            _lib.check(_lib.load().kpm_run_set_probes(self._h, _lib.ptr(z), z.shape[1]),
                       "run_set_probes")

    def set_probe_block(self, z, ldz):
        """z: host ndarray or device pointer (int), n x k with row stride ldz."""
        _lib.check(_lib.load().kpm_run_set_probes(self._h, _lib.ptr(z), int(ldz)),
                   "run_set_probes")

    def advance(self, steps=None) -> int:
        rem = ctypes.c_int32()
        s = self.total_steps if steps is None else int(steps)
        _lib.check(_lib.load().kpm_run_advance(self._h, s, ctypes.byref(rem)), "run_advance")
        return rem.value

    def result(self, out, trace_scale=1.0):
        bad = ctypes.c_int64(-1)
        _lib.check(_lib.load().kpm_run_result(self._h, _lib.ptr(out), float(trace_scale),
                                              ctypes.byref(bad)), "run_result")
        return out

    def set_timing(self, enable=True):
        _lib.check(_lib.load().kpm_run_set_timing(self._h, 1 if enable else 0))

    def kernel_time(self):
        """(summed step-kernel milliseconds, launches) since the last call."""
        ms, n = ctypes.c_double(), ctypes.c_int32()
        _lib.check(_lib.load().kpm_run_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def block(self):
        """(device pointer of T_k, row stride, k) for bit-exactness checks."""
        p, ld, ki = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int32()
        _lib.check(_lib.load().kpm_run_block(self._h, ctypes.byref(p), ctypes.byref(ld),
                                             ctypes.byref(ki)))
        return p.value, ld.value, ki.value

    def free(self):
        if self._h is not None:
            _lib.load().kpm_run_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _batch_cols(dev, nz, blocks, max_cols=1024, fixed_bytes=0):
    """Probe columns per batch: all of them when two/three n x ld fp64 blocks
    (plus `fixed_bytes` of per-run buffers, e.g. the (n, M+1) LDOS result)
    fit in 85% of free HBM, else the largest multiple of 32 that does."""
    dev.prepare(min(nz, max_cols, 128))  # the twin (if any) exists before free memory is read
    free, _ = dev.ctx.mem_info()
    per_col = 8 * max(dev.n, 1) * blocks
    fit = int(max(0.85 * free - fixed_bytes, 0) // per_col)
    b = min(nz, max_cols, max(fit, 1))
    if b < nz and b > 32:
        b -= b % 32
    return max(1, b)


def _shards(nz, ctxs):
    """Contiguous balanced column ranges, one per context (empty ones dropped)."""
    out = []
    base, extra = divmod(nz, len(ctxs))
    c0 = 0
    for i, ctx in enumerate(ctxs):
        c1 = c0 + base + (1 if i < extra else 0)
        if c1 > c0:
            out.append((ctx, c0, c1))
        c0 = c1
    return out


def _fan_out(jobs):
    """Run one job per GPU context on its own host thread (the C-ABI calls
    release the GIL); re-raise the first failure."""
    if len(jobs) == 1:
        return [jobs[0]()]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(jobs)) as ex:
        futs = [ex.submit(j) for j in jobs]
        return [f.result() for f in futs]


def _contexts(dev, threads):
    """GPU contexts of one call: the graph's own context alone, or the pool of
    _lib.devices_for(threads) (the graph is replicated where needed)."""
    devs = _lib.devices_for(threads)
    return [dev.ctx] if len(devs) <= 1 else _lib.Context.pool(devs)


def dos_contrib(sop, probes: ProbeMatrix, m_max: int, doubling=True, batch=None, threads=1):
    """Per-probe contribution matrix contrib[m, j] = z_j^T T_m z_j, shape
    (m_max+1, nz) (kpm.py:104-108), computed on the device.  With several
    GPUs (``threads`` / KPM_DEVICES, see _lib.devices_for) each takes a
    contiguous column range on a replica of the graph; the columns are
    independent and their sums fixed by the graph alone, so the result is
    bitwise that of one GPU and needs no collective."""
    dev = _device_graph(sop)
    nz = probes.nz
    contrib = np.empty((m_max + 1, nz))
    mode = _lib.MODE_DOS_DOUBLING if doubling else _lib.MODE_DOS_DIRECT

    def job(ctx, a0, a1):
        g = dev.on(ctx)
        b = batch or _batch_cols(g, a1 - a0, 2 if doubling else 3)
        for c0 in range(a0, a1, b):
            c1 = min(a1, c0 + b)
            sub = probes.column_slice(c0, c1) if (c0, c1) != (0, nz) else probes
            run = Run(g, c1 - c0, mode, m_max)
            try:
                run.set_probes(sub)
                run.advance()
                part = np.empty((m_max + 1, c1 - c0))
                run.result(part)
            finally:
                run.free()
            contrib[:, c0:c1] = part

    _fan_out([lambda c=c, a=a, b=b: job(c, a, b)
              for c, a, b in _shards(nz, _contexts(dev, threads))])
    return contrib


def dos_moments(sop, probes: ProbeMatrix, m_max: int, effective_dim=None, threads=1,
                doubling=True, batch=None) -> ChebMoments:
    """Global moments d_m = tr(T_m(H))/N by stochastic trace estimation
    (kpm.py:92-117).  ``doubling`` (default) evaluates the M+1 moments from
    ceil(M/2) recurrence steps via T_2k = 2T_k^2 - I, T_2k+1 = 2T_k+1 T_k - T_1;
    ``doubling=False`` is the reference's direct estimator z^T T_m z.
    ``threads`` > 1 spreads the probe columns over that many GPUs
    (_lib.devices_for)."""
    if m_max < 0:
        raise ValueError("m_max must be >= 0")
    if sop.n != probes.n:
        raise ValueError("probe dimension does not match operator")
    denom = float(effective_dim) if effective_dim is not None else float(sop.n)
    contrib = dos_contrib(sop, probes, m_max, doubling=doubling, batch=batch, threads=threads)
    if not np.all(np.isfinite(contrib)):
        raise RecurrenceBlowupError(_BLOWUP)
    values = contrib.sum(axis=1) * (probes.trace_scale / denom)
    return ChebMoments(mode=MODE_GLOBAL, values=values, scale_map=sop.scale_map,
                       probe_meta=probes.meta())


def _ldos_run(sop, probes: ProbeMatrix, m_max: int, flags, batch=None, threads=1):
    """A finished-steps LDOS run holding the per-node sums over ALL probe
    columns (kpm.py:133-144): each GPU runs its column shard in batches,
    batches and shards are added into the first run on the device
    (kpm_run_accumulate: same-GPU add, or a peer copy from another GPU), so
    the (n, M+1) block never round-trips through the host.  The caller owns
    the returned Run (result() then free())."""
    dev = _device_graph(sop)
    n, nz = sop.n, probes.nz
    lib = _lib.load()
    ldos_bytes = 8 * n * (m_max + 1)

    def job(ctx, a0, a1):
        g = dev.on(ctx)
        b = batch or _batch_cols(g, a1 - a0, 3, max_cols=1 << 30, fixed_bytes=ldos_bytes)
        if b < a1 - a0 and not batch:  # an accumulator run sits beside each batch
            b = _batch_cols(g, a1 - a0, 3, max_cols=1 << 30, fixed_bytes=2 * ldos_bytes)
        acc = None
        try:
            for c0 in range(a0, a1, b):
                c1 = min(a1, c0 + b)
                sub = probes.column_slice(c0, c1) if (c0, c1) != (0, nz) else probes
                run = Run(g, c1 - c0, _lib.MODE_LDOS, m_max, flags)
                try:
                    run.set_probes(sub)
                    run.advance()  # queued: the caller's host work overlaps
                    if acc is None:
                        if c1 < a1:  # more batches follow: keep only the sums
                            _lib.check(lib.kpm_run_trim(run._h), "run_trim")
                        acc, run = run, None
                    else:
                        _lib.check(lib.kpm_run_accumulate(acc._h, run._h), "run_accumulate")
                finally:
                    if run is not None:
                        run.free()
        except BaseException:
            if acc is not None:
                acc.free()
            raise
        return acc

    runs = _fan_out([lambda c=c, a=a, b=b: job(c, a, b)
                     for c, a, b in _shards(nz, _contexts(dev, threads))])
    try:
        for other in runs[1:]:
            _lib.check(lib.kpm_run_accumulate(runs[0]._h, other._h), "run_accumulate")
    except BaseException:
        for r in runs:
            r.free()
        raise
    for other in runs[1:]:
        other.free()
    return runs[0]


def pdos_num(sop, probes: ProbeMatrix, m_max: int, threads=1) -> np.ndarray:
    """Raw per-node sums num[i, m] = sum_j z_ij (T_m z)_ij, shape (n, m_max+1)
    (kpm.py:135-136, node-major) -- the quantity sharded runs all-reduce."""
    run = _ldos_run(sop, probes, m_max, _lib.LDOS_RAW, threads=threads)
    try:
        out = np.empty((sop.n, m_max + 1))
        run.result(out, 1.0)
    finally:
        run.free()
    return out


def pdos_moments(sop, probes: ProbeMatrix, m_max: int, normalized=True, threads=1,
                 batch=None) -> ChebMoments:
    """Per-node moments c_mk ~= T_m(H)_kk (kpm.py:120-152): the fused kernel
    reduces z (.) T_m z across each row's probe columns every step and writes
    the (n, M+1) result in place; probe batches and GPU shards (``threads``)
    are summed on the device before the normalisation."""
    if m_max < 0:
        raise ValueError("m_max must be >= 0")
    if sop.n != probes.n:
        raise ValueError("probe dimension does not match operator")
    run = _ldos_run(sop, probes, m_max, 0 if normalized else _lib.LDOS_RAW, batch=batch,
                    threads=threads)
    try:
        values = np.empty((sop.n, m_max + 1))
        _lib.prefault(values)
        run.result(values, probes.trace_scale)
    finally:
        run.free()
    return ChebMoments(mode=MODE_PER_NODE, values=values, scale_map=sop.scale_map,
                       probe_meta=probes.meta())
