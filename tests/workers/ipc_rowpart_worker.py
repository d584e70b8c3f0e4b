"""Worker of tests/test_gpu_ipc_partition.py: one of WORLD processes, all on
cuda:0, gloo for the control plane (barriers / object all-gathers on the host;
no kernel waits on another process's kernel).  Rank r owns a row range of an
R-MAT graph; the fused step kernel gathers the peers' rows through CUDA IPC
mappings of their recurrence blocks (distributed.dos_moments_row_partitioned).
Rank 0 compares with the unpartitioned run and writes the verdict."""

import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import torch.distributed as dist  # noqa: E402

import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import distributed as kdist  # noqa: E402
from paper_1905_09758_b200 import partition  # noqa: E402


def main():
    out = sys.argv[1]
    scale, ef, seed, nz, m_max = 13, 16, 2, 40, 30
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    n = 1 << scale
    full = kp.DeviceGraph.rmat(scale, ef, seed)
    rp, _, _ = full.export()
    bounds = [int(b) for b in partition.balanced_bounds(rp, world)]
    part = partition.part_rmat(scale, ef, seed, bounds[rank], bounds[rank + 1])
    probes = kp.make_probes(n, nz, "rademacher", seed=seed)  # device-generated rows
    res = {}
    for doubling in (False, True):
        mom = kdist.dos_moments_row_partitioned(part, bounds, probes, m_max, doubling=doubling)
        if rank == 0:
            sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(full), (-1.0, 1.0))
            want = kp.dos_moments(sop, probes, m_max, doubling=doubling)
            err = float(np.max(np.abs(mom.values - want.values)) / np.max(np.abs(want.values)))
            res["doubling" if doubling else "direct"] = err
    # explicit host probe block: each rank uploads its own rows
    z = np.random.default_rng(5).standard_normal((n, 6))
    pm = kp.ProbeMatrix(n, 6, "gaussian", 5, columns=z)
    mom = kdist.dos_moments_row_partitioned(part, bounds, pm, 12, doubling=False)
    if rank == 0:
        sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(full), (-1.0, 1.0))
        want = kp.dos_moments(sop, pm, 12, doubling=False)
        res["host_block"] = float(np.max(np.abs(mom.values - want.values))
                                  / np.max(np.abs(want.values)))
        res["world"] = world
        res["bounds"] = bounds
        with open(out, "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
