"""The N>1 probe-sharded path on CPU: world_size-2 gloo process groups.

Each rank computes its column range of the per-probe contribution matrix (the
oracle stands in for the device kernel here -- these tests cover the host
plumbing: sharding, zero-padded all-reduce, final scaling) and the result must
equal the single-process answer bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1905_09758_b200 as kp
        from oracle import netdos_oracle as orc
        from paper_1905_09758_b200.distributed import (dos_moments_sharded,
                                                       pdos_moments_sharded)

        g = kp.erdos_renyi(300, 0.03, seed=2)
        sop = kp.scaled_operator_for(g, "normalized-adjacency")
        data = orc.normadj_values(g.row_ptr, g.col_idx)

        def contrib_fn(s, p, m, doubling=True):
            return orc.c_dos_contrib(g.row_ptr, g.col_idx, data, p.columns, m)

        def num_fn(s, p, m):
            return np.ascontiguousarray(orc.c_ldos_num(g.row_ptr, g.col_idx, data,
                                                       p.columns, m).T)

        probes = kp.make_probes(g.n, 13, "rademacher", seed=4)
        d = dos_moments_sharded(sop, probes, 40, contrib_fn=contrib_fn)
        pd = pdos_moments_sharded(sop, probes, 12, num_fn=num_fn)
        if rank == 0:
            out["dos"] = d.values
            out["pdos"] = pd.values
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_process():
    import paper_1905_09758_b200 as kp
    from oracle import netdos_oracle as orc

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)

    g = kp.erdos_renyi(300, 0.03, seed=2)
    data = orc.normadj_values(g.row_ptr, g.col_idx)
    z = kp.make_probes(g.n, 13, "rademacher", seed=4).columns
    contrib = orc.c_dos_contrib(g.row_ptr, g.col_idx, data, z, 40)
    want = contrib.sum(axis=1) * ((1.0 / 13) / g.n)
    assert np.array_equal(out["dos"], want)
    num = orc.c_ldos_num(g.row_ptr, g.col_idx, data, z, 12)
    want_p = (num / num[0]).T
    assert np.max(np.abs(out["pdos"] - want_p)) < 1e-13


@pytest.mark.parametrize("world", [2, 3])
def test_column_slices_partition_the_probe_family(world):
    import paper_1905_09758_b200 as kp
    from paper_1905_09758_b200.distributed import shard_range

    p = kp.make_probes(50, 10, "rademacher", seed=3)
    full = kp.make_probes(50, 10, "rademacher", seed=3).columns
    parts = [p.column_slice(*shard_range(10, r, world)).columns for r in range(world)]
    assert np.array_equal(np.concatenate(parts, axis=1), full)


def test_row_partition_raw_sums_and_doubling_transform(oracle):
    """Host side of the row-partitioned path: per-partition raw doubling sums
    (<T_s,T_s-1>, <T_s,T_s>), added in partition order, then the doubling
    transform == the direct estimator z^T T_m z (oracle) to rounding."""
    import paper_1905_09758_b200 as kp
    from paper_1905_09758_b200.partition import balanced_bounds, doubling_transform

    g = kp.erdos_renyi(400, 0.02, seed=3)
    data = oracle.normadj_values(g.row_ptr, g.col_idx)
    z = kp.make_probes(g.n, 6, "rademacher", seed=1).columns
    M = 20
    blocks = [z] + [oracle.c_recurrence_block(g.row_ptr, g.col_idx, data, z, s)
                    for s in range(1, M // 2 + 1)]
    bounds = balanced_bounds(g.row_ptr, 3)
    raw = np.zeros((M + 1, 6))
    for q in range(3):
        lo, hi = bounds[q], bounds[q + 1]
        part = np.zeros((M + 1, 6))
        part[0] = np.einsum("ij,ij->j", z[lo:hi], z[lo:hi])
        for s in range(1, M // 2 + 1):
            t, tp = blocks[s][lo:hi], blocks[s - 1][lo:hi]
            part[2 * s - 1] = np.einsum("ij,ij->j", t, tp)
            part[2 * s] = np.einsum("ij,ij->j", t, t)
        raw += part
    got = doubling_transform(raw, M)
    want = oracle.c_dos_contrib(g.row_ptr, g.col_idx, data, z, M)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
