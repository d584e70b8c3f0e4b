#!/usr/bin/env python3
"""Bandwidth over time of one traced step launch (KPM_TRACE dump): per 1/40 of
the span, the bytes the active work items stand for (512 B per nonzero of a
64-column tile + 3 x 512 B per row), spread uniformly over each item's
duration -- shows whether the tail of short / empty rows runs below the
gather-heavy body."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from trace_report import load  # noqa: E402


def main(path, seg_bytes):
    nh_tasks, n_chunks, ld, n_heavy, tr, co, cst = load(path)
    t0 = tr[:, 0].astype(np.int64)
    t1 = tr[:, 1].astype(np.int64)
    base = t0.min()
    s, e = (t0 - base) / 1e6, (t1 - base) / 1e6
    span = e.max()
    lid = np.arange(nh_tasks, len(s))
    ch = co[lid - nh_tasks]
    rows, nnz, empty = cst[ch, 0], cst[ch, 1], cst[ch, 2]
    bytes_item = nnz * seg_bytes + rows * 3 * seg_bytes
    nb = 40
    edges = np.linspace(0, span, nb + 1)
    bw = np.zeros(nb)
    rows_t = np.zeros(nb)
    nnz_t = np.zeros(nb)
    for k in range(nb):
        a, b = edges[k], edges[k + 1]
        ov = np.clip(np.minimum(e[lid], b) - np.maximum(s[lid], a), 0, None)
        frac = ov / np.maximum(e[lid] - s[lid], 1e-9)
        bw[k] = (bytes_item * frac).sum() / ((b - a) * 1e-3) / 1e12
        rows_t[k] = (rows * frac).sum()
        nnz_t[k] = (nnz * frac).sum()
    out = {"file": path, "span_ms": round(float(span), 3), "items": int(len(s)),
           "rows_total": int(rows.sum()), "empty_rows": int(empty.sum()),
           "model_TBps_per_window": [round(float(x), 2) for x in bw],
           "avg_degree_per_window": [round(float(n_ / max(r_, 1)), 1) for n_, r_ in zip(nnz_t, rows_t)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 512)
