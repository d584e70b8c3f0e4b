"""Probe sharding across GPUs: one process per GPU.

Probe columns are independent units: rank r of N takes the contiguous column
range [r*P/N, (r+1)*P/N), the CSR is replicated on every GPU, and the only
exchange is ONE all-reduce (sum, fp64) of the zero-padded (M+1) x P
per-probe contribution matrix -- every column is written by exactly one rank,
so the sum is exact and the host finishes identically to 1 GPU.  LDOS sums
per-node numerators with one all-reduce of the (n, M+1) block.

torch.distributed (NCCL on B200, gloo in the CPU tests) is plumbing only.
"""

from __future__ import annotations

import numpy as np

from .errors import RecurrenceBlowupError
from .kpm import _BLOWUP, MODE_GLOBAL, MODE_PER_NODE, ChebMoments


def shard_range(nz: int, rank: int, world: int):
    """Contiguous, balanced column range of `rank` (sizes differ by <= 1)."""
    base, extra = divmod(nz, world)
    c0 = rank * base + min(rank, extra)
    return c0, c0 + base + (1 if rank < extra else 0)


def _allreduce_sum(arr: np.ndarray, group=None) -> np.ndarray:
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    if backend == "nccl":
        t = torch.from_numpy(arr).cuda()
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().numpy()
    t = torch.from_numpy(arr)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.numpy()


def _backend(group):
    import torch.distributed as dist

    return dist.get_backend(group)


def _world(group):
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def combine_contrib(local: np.ndarray, c0: int, nz: int, group=None) -> np.ndarray:
    """Zero-pad this rank's (M+1) x (c1-c0) block into (M+1) x nz and sum."""
    full = np.zeros((local.shape[0], nz))
    full[:, c0:c0 + local.shape[1]] = local
    _, world = _world(group)
    return _allreduce_sum(full, group) if world > 1 else full


def dos_moments_sharded(sop, probes, m_max, effective_dim=None, doubling=True,
                        group=None, contrib_fn=None) -> ChebMoments:
    """dos_moments with probe columns sharded over the process group."""
    rank, world = _world(group)
    c0, c1 = shard_range(probes.nz, rank, world)
    if contrib_fn is None:
        from .kpm import dos_contrib as contrib_fn
    local = contrib_fn(sop, probes.column_slice(c0, c1), m_max, doubling=doubling) \
        if c1 > c0 else np.zeros((m_max + 1, 0))
    contrib = combine_contrib(local, c0, probes.nz, group)
    if not np.all(np.isfinite(contrib)):
        raise RecurrenceBlowupError(_BLOWUP)
    denom = float(effective_dim) if effective_dim is not None else float(sop.n)
    values = contrib.sum(axis=1) * (probes.trace_scale / denom)
    return ChebMoments(mode=MODE_GLOBAL, values=values, scale_map=sop.scale_map,
                       probe_meta=probes.meta())


def _device_num_allreduce(sop, sub, m_max, group):
    """NCCL path: this rank's raw per-node sums land in a CUDA tensor straight
    from the run's device buffer (D2D) and are summed in place by one
    all-reduce over NVLink -- no host round trip of the (n, M+1) block."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .kpm import _device_graph, _ldos_run

    dev = _device_graph(sop)
    num = torch.zeros((sop.n, m_max + 1), dtype=torch.float64,
                      device=torch.device("cuda", dev.ctx.device))
    if sub is not None:
        run = _ldos_run(sop, sub, m_max, _lib.LDOS_RAW)
        try:
            run.result(num.data_ptr(), 1.0)  # synchronous on the library stream
        finally:
            run.free()
    dist.all_reduce(num, op=dist.ReduceOp.SUM, group=group)
    return num


def pdos_moments_sharded(sop, probes, m_max, normalized=True, group=None,
                         num_fn=None) -> ChebMoments:
    """pdos_moments with probe columns sharded: per-node raw sums all-reduced
    (NCCL: on the device; gloo: host arrays), then kpm.py:143-151."""
    rank, world = _world(group)
    c0, c1 = shard_range(probes.nz, rank, world)
    sub = probes.column_slice(c0, c1) if c1 > c0 else None
    if num_fn is None and world > 1 and _backend(group) == "nccl":
        t = _device_num_allreduce(sop, sub, m_max, group)
        if not bool(t.isfinite().all()):
            raise RecurrenceBlowupError(_BLOWUP)
        if normalized:
            den = t[:, 0]
            zero = (den == 0.0).nonzero()
            if zero.numel():
                raise ValueError(f"zero probe mass at node {int(zero[0, 0])}; "
                                 "its moments are unrecoverable")
            t = t / den[:, None]  # IEEE division, as numpy's (num / den).T
        else:
            t = t * probes.trace_scale
        return ChebMoments(mode=MODE_PER_NODE, values=t.cpu().numpy(),
                           scale_map=sop.scale_map, probe_meta=probes.meta())
    if num_fn is None:
        from .kpm import pdos_num as num_fn
    local = num_fn(sop, sub, m_max) if sub is not None else np.zeros((sop.n, m_max + 1))
    num = _allreduce_sum(np.ascontiguousarray(local), group) if world > 1 else local
    if not np.all(np.isfinite(num)):
        raise RecurrenceBlowupError(_BLOWUP)
    if normalized:
        den = num[:, 0].copy()
        if np.any(den == 0.0):
            k = int(np.argmax(den == 0.0))
            raise ValueError(f"zero probe mass at node {k}; its moments are unrecoverable")
        values = num / den[:, None]
    else:
        values = num * probes.trace_scale
    return ChebMoments(mode=MODE_PER_NODE, values=np.ascontiguousarray(values),
                       scale_map=sop.scale_map, probe_meta=probes.meta())


def broadcast_graph(dev, group=None, src=0, ctx=None):
    """Replicate a device graph to every rank of an NCCL group: rank `src`
    holds `dev` (e.g. loaded once from the host), the others pass None; the
    int64 row_ptr and int32 col_idx go out in two NCCL broadcasts over
    NVLink/NVSwitch and each rank rebuilds d^-1/2 and its schedule from them
    (bit-identical).  Replaces N host loads/uploads of the same CSR
    (the CSR is replicated per GPU)."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .graph import DeviceGraph

    rank, world = _world(group)
    if world <= 1:
        return dev
    ctx = ctx or (dev.ctx if dev is not None else _lib.Context.get())
    cuda = torch.device("cuda", ctx.device)
    meta = torch.zeros(3, dtype=torch.int64, device=cuda)
    if rank == src:
        if dev.explicit:
            raise ValueError("broadcast_graph replicates implicit (unit-weight) graphs")
        meta[0], meta[1] = dev.n, dev.nnz
    dist.broadcast(meta, src, group=group)
    n, nnz = int(meta[0]), int(meta[1])
    rp = torch.empty(n + 1, dtype=torch.int64, device=cuda)
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=cuda)
    if rank == src:
        _lib.check(_lib.load().kpm_graph_export(dev.handle, rp.data_ptr(), ci.data_ptr(),
                                                None), "graph_export")
    dist.broadcast(rp, src, group=group)
    dist.broadcast(ci, src, group=group)
    torch.cuda.synchronize(cuda)
    if rank != src:
        dev = DeviceGraph.from_csr(n, rp.data_ptr(), (ci.data_ptr(), nnz, "int32"), ctx=ctx)
    del rp, ci
    return dev


# ------------------------------------------------ row-partitioned (§8e) ---
def _all_gather_arrays(arr: np.ndarray, group=None):
    """All-gather variable-length 1-D float64 arrays (rank order)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, np.ascontiguousarray(arr), group=group)
    return out


def dos_moments_row_partitioned(part, bounds, probes, m_max, effective_dim=None,
                                doubling=True, group=None):
    """Global moments with rank r owning rows [bounds[r], bounds[r+1]) of H.

    ``part`` is this rank's partition (``partition.part_rmat`` /
    ``partition.part_from_csr``).  Each rank exports the CUDA IPC handles of
    its two recurrence blocks; every rank maps all peers' blocks, so the fused
    step kernel gathers remote rows straight from peer HBM over NVLink /
    NVSwitch.  Ranks barrier between steps (a rank overwrites its T_{k-1}
    block in step k+1 only after every peer finished gathering T_k)."""
    import ctypes

    import torch.distributed as dist

    from . import _lib
    from .kpm import Run
    from .partition import doubling_transform

    rank, world = _world(group)
    lib = _lib.load()
    dinv_parts = _all_gather_arrays(part.export()[2], group)
    part.set_dinv(np.concatenate(dinv_parts))
    mode = _lib.MODE_DOS_DOUBLING if doubling else _lib.MODE_DOS_DIRECT
    run = Run(part, probes.nz, mode, m_max)
    opened = []
    try:
        if probes.device_generated:
            run.set_probes(probes)
        else:
            z = np.ascontiguousarray(probes.columns[bounds[rank]:bounds[rank + 1]])
            run.set_probe_block(z, z.shape[1])
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(lib.kpm_run_blocks(run._h, ctypes.byref(a), ctypes.byref(b)))
        ha, hb = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
        _lib.check(lib.kpm_ipc_get_handle(a, ha), "ipc_get_handle")
        _lib.check(lib.kpm_ipc_get_handle(b, hb), "ipc_get_handle")
        handles = [None] * world
        dist.all_gather_object(handles, (ha.raw, hb.raw), group=group)
        pa, pb = [], []
        for q, (qa, qb) in enumerate(handles):
            if q == rank:
                pa.append(a.value)
                pb.append(b.value)
                continue
            for raw, dst in ((qa, pa), (qb, pb)):
                p = ctypes.c_void_p()
                _lib.check(lib.kpm_ipc_open_handle(part.ctx.handle,
                                                   ctypes.create_string_buffer(raw, 64),
                                                   ctypes.byref(p)), "ipc_open_handle")
                opened.append(p.value)
                dst.append(p.value)
        lo = np.ascontiguousarray(bounds, dtype=np.int64)
        arr_a = (ctypes.c_void_p * world)(*pa)
        arr_b = (ctypes.c_void_p * world)(*pb)
        _lib.check(lib.kpm_run_set_partition(run._h, world, _lib.ptr(lo), rank,
                                             ctypes.cast(arr_a, ctypes.c_void_p),
                                             ctypes.cast(arr_b, ctypes.c_void_p)),
                   "run_set_partition")
        dist.barrier(group=group)
        for _ in range(run.total_steps):
            run.advance(1)
            part.ctx.synchronize()
            dist.barrier(group=group)
        raw = np.empty((m_max + 1, probes.nz))
        run.result(raw)
    finally:
        for p in opened:
            lib.kpm_ipc_close(p)
        run.free()
    parts = [None] * world
    dist.all_gather_object(parts, raw, group=group)
    total = np.zeros_like(raw)
    for x in parts:  # rank order: deterministic for a fixed partition
        total += x
    contrib = doubling_transform(total, m_max) if doubling else total
    if not np.all(np.isfinite(contrib)):
        raise RecurrenceBlowupError(_BLOWUP)
    denom = float(effective_dim) if effective_dim is not None else float(bounds[-1])
    from .operators import IDENTITY_MAP
    return ChebMoments(mode=MODE_GLOBAL, values=contrib.sum(axis=1) * (probes.trace_scale / denom),
                       scale_map=IDENTITY_MAP, probe_meta=probes.meta())
