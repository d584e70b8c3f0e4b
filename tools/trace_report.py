#!/usr/bin/env python3
"""Summarise a KPM_TRACE dump of one fused-step launch: kernel span, when the
work queue ran dry, the tail, and the slowest work items (hub slices vs light
chunks, with the chunk's rows / nonzeros / isolated rows)."""
import json
import sys

import numpy as np


def load(path):
    raw = open(path, "rb").read()
    nh_tasks, n_chunks, ld, n_heavy = np.frombuffer(raw[:32], dtype=np.int64)
    items = nh_tasks + n_chunks
    off = 32
    tr = np.frombuffer(raw[off:off + 24 * items], dtype=np.uint64).reshape(items, 3)
    off += 24 * items
    co = np.frombuffer(raw[off:off + 4 * n_chunks], dtype=np.int32)
    off += 4 * n_chunks
    cst = np.frombuffer(raw[off:off + 24 * n_chunks], dtype=np.int64).reshape(n_chunks, 3)
    return int(nh_tasks), int(n_chunks), int(ld), int(n_heavy), tr, co, cst


def report(path):
    nh_tasks, n_chunks, ld, n_heavy, tr, co, cst = load(path)
    t0 = tr[:, 0].astype(np.int64)
    t1 = tr[:, 1].astype(np.int64)
    base = t0.min()
    s, e = (t0 - base) / 1e6, (t1 - base) / 1e6  # ms
    dur = e - s
    span = e.max()
    heavy = np.arange(len(s)) < nh_tasks
    out = {"file": path, "ld": ld, "items": len(s), "hub_tasks": nh_tasks,
           "span_ms": round(float(span), 3),
           "queue_dry_ms": round(float(s.max()), 3),
           "hub_task_ms_max": round(float(dur[heavy].max()), 3) if nh_tasks else 0,
           "hub_task_ms_sum": round(float(dur[heavy].sum()), 3) if nh_tasks else 0,
           "light_ms_mean": round(float(dur[~heavy].mean()), 4),
           "light_ms_max": round(float(dur[~heavy].max()), 3)}
    # busy warps over time (fraction of the span with >= 90% of warps busy)
    ev = np.concatenate([np.stack([s, np.ones_like(s)], 1), np.stack([e, -np.ones_like(e)], 1)])
    ev = ev[np.argsort(ev[:, 0], kind="stable")]
    busy = np.cumsum(ev[:, 1])
    peak = busy.max()
    dt = np.diff(ev[:, 0], append=ev[-1, 0])
    out["warps_peak"] = int(peak)
    out["warp_util"] = round(float((busy * dt).sum() / (peak * span)), 3)
    for q in (0.5, 0.9):
        # time when busy first drops below q*peak for good
        below = np.where(busy < q * peak)[0]
        last_above = np.where(busy >= q * peak)[0]
        out[f"t_last_busy{int(q*100)}_ms"] = round(float(ev[last_above.max(), 0]), 3) if len(last_above) else 0
    # light chunk stats
    lid = np.arange(nh_tasks, len(s))
    ch = co[lid - nh_tasks]
    rows, nnz, empty = cst[ch, 0], cst[ch, 1], cst[ch, 2]
    slow = np.argsort(-dur[lid])[:12]
    out["slowest_light"] = [
        {"item": int(lid[k]), "start": round(float(s[lid[k]]), 3), "ms": round(float(dur[lid[k]]), 3),
         "rows": int(rows[k]), "nnz": int(nnz[k]),
         "empty_rows": int(empty[k])}
        for k in slow]
    last = np.argsort(-e)[:8]
    out["last_finishing"] = [{"item": int(k), "hub": bool(heavy[k]), "start": round(float(s[k]), 3),
                              "end": round(float(e[k]), 3)} for k in last]
    # per-chunk time model: ms vs (rows, nnz)
    A = np.stack([rows - empty, empty, nnz, np.ones_like(rows)], 1).astype(float)
    coef, *_ = np.linalg.lstsq(A, dur[lid], rcond=None)
    out["fit_us_per_row_emptyrow_nnz_const"] = [round(float(c) * 1e3, 5) for c in coef]
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps(report(p)))
