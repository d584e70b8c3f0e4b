#!/usr/bin/env python3
"""Experiment: does a degree-descending relabelling (hot rows contiguous at
the start of every recurrence block) plus a persisting L2 access-policy
window over those rows (KPM_WINDOW_MB) lower the DRAM traffic / step time of
the fused step on C5?  The relabelled CSR is built with torch on the device
(row order by degree desc, ids mapped; neighbour order not preserved -- a
performance experiment only, results are not parity-checked).

    KPM_WINDOW_MB=79 python tools/r2/relabel_exp.py --probes 32 128 [--only relab]
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402
from paper_1905_09758_b200.kpm import Run  # noqa: E402


def relabel(dev):
    n, nnz = dev.n, dev.nnz
    cuda = torch.device("cuda", dev.ctx.device)
    rp = torch.empty(n + 1, dtype=torch.int64, device=cuda)
    ci = torch.empty(nnz, dtype=torch.int32, device=cuda)
    _lib.check(_lib.load().kpm_graph_export(dev.handle, rp.data_ptr(), ci.data_ptr(), None))
    deg = rp[1:] - rp[:-1]
    order = torch.argsort(-deg, stable=True)  # new id -> old id
    inv = torch.empty_like(order)
    inv[order] = torch.arange(n, device=cuda)
    nd = deg[order]
    rp2 = torch.zeros(n + 1, dtype=torch.int64, device=cuda)
    rp2[1:] = torch.cumsum(nd, 0)
    offs = rp[:-1][order] - rp2[:-1]
    ci2 = torch.empty_like(ci)
    step = 1 << 28
    rows_of = torch.repeat_interleave(torch.arange(n, device=cuda), nd, output_size=nnz)
    for a in range(0, nnz, step):
        b = min(nnz, a + step)
        pos = torch.arange(a, b, device=cuda, dtype=torch.int64) + offs[rows_of[a:b]]
        ci2[a:b] = inv[ci[pos].long()].int()
    del ci, rp, offs, inv, order
    if os.environ.get("KPM_EXP_SORT", "1") == "1":
        # canonical CSR of the relabelled graph: each row sorted by new id,
        # i.e. by degree descending -- the hot neighbours first
        key = rows_of * n + ci2.long()
        del rows_of
        key = torch.sort(key)[0]
        ci2 = (key % n).int()
        del key
    else:
        del rows_of
    torch.cuda.synchronize()
    g2 = kp.DeviceGraph.from_csr(n, rp2.data_ptr(), (ci2.data_ptr(), nnz, "int32"), ctx=dev.ctx)
    del rp2, ci2
    torch.cuda.empty_cache()
    return g2


def time_steps(dev, P, steps=6, warmup=3):
    run = Run(dev, P, _lib.MODE_DOS_DOUBLING, 2 * (steps + warmup) + 2)
    run.set_probes(kp.make_probes(dev.n, P, "rademacher", seed=4))
    run.advance(warmup)
    dev.ctx.synchronize()
    run.set_timing(True)
    run.advance(steps)
    ms, nl = run.kernel_time()
    run.free()
    return ms / nl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--probes", type=int, nargs="+", default=[32, 128])
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--only", default="")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--hotk", type=int, nargs="+", default=[0])
    a = ap.parse_args()
    ctx = _lib.Context.get(0)
    dev = kp.DeviceGraph.rmat(a.scale, 16, 4, ctx=ctx)
    t0 = time.time()
    g2 = relabel(dev)
    t_rel = time.time() - t0
    graphs = {"orig": dev, "relab": g2}
    for name, g in graphs.items():
        if a.only and name != a.only:
            continue
        for P in a.probes:
            for hotk in (a.hotk if name == "relab" else [0]):
                os.environ["KPM_EXP_HOTK"] = str(hotk)
                ms = time_steps(g, P, a.steps)
                print(json.dumps({"graph": name, "P": P, "hotk": hotk, "ms_per_step": round(ms, 2),
                                  "window_mb": os.environ.get("KPM_WINDOW_MB", "0"),
                                  "g4hot": os.environ.get("KPM_G4_HOT", "default"),
                                  "relabel_s": round(t_rel, 2)}), flush=True)


if __name__ == "__main__":
    main()
