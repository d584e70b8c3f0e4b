#!/usr/bin/env python3
"""Graph-file fixtures for the device ingest path,
with the expected results written BY THE REFERENCE's own parse_graph_file
(fileio.py:104-128) -- run only in the build container, where
/root/reference exists.  Writes tests/golden/files/* and
tests/golden/fileio.json; paths in error messages are stored as "{path}".

    python tests/golden/make_fileio_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
FILES = os.path.join(HERE, "files")
sys.path.insert(0, REPO)

from oracle import netdos_oracle as orc  # noqa: E402

assert orc.ref_spmv() is not None, "run `make -C oracle` first"
sys.path.insert(0, "/root/reference/pkg/src")
from netdos import parse_graph_file  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_edgelist(seed, n_lines, id_space, comment_every=97, weighted=False):
    rng = np.random.default_rng(seed)
    ids = rng.choice(id_space, size=max(2, id_space // 3), replace=False) - id_space // 5
    out = ["# random edge list, seed %d" % seed]
    seen = set()
    k = 0
    while k < n_lines:
        a, b = (int(x) for x in rng.choice(ids, 2))
        if a == b or (a, b) in seen:
            continue
        seen.add((a, b))
        seen.add((b, a)) if rng.random() < 0.9 else None
        sep = ["\t", " ", "  "][k % 3]
        line = f"{a}{sep}{b}"
        if weighted:
            line += f" {rng.integers(1, 9) / 4}"
        if k % 11 == 0:
            line += "   "
        out.append(line)
        if k % comment_every == 0:
            out.append("% a comment" if k % 2 else "")
        k += 1
    return "\n".join(out) + "\n"


def random_mm(seed, n, nnz):
    rng = np.random.default_rng(seed)
    pairs = set()
    while len(pairs) < nnz:
        i, j = (int(x) for x in rng.integers(1, n + 1, 2))
        if i != j:
            pairs.add((max(i, j), min(i, j)))
    lines = ["%%MatrixMarket matrix coordinate pattern symmetric", "% generated",
             f"{n} {n} {nnz}"]
    lines += [f"{i} {j}" for i, j in sorted(pairs)]
    return "\n".join(lines) + "\n"


CASES = {
    # name: (file name, bytes/text, kwargs)
    "comments": ("comments.txt", "# comment\n0 1\n1 2\n", {}),
    "weighted": ("weighted.txt", "0 1 2.5\n", {}),
    "sparse_ids": ("sparse_ids.txt", "% comment\n5 9\n9 70\n", {}),
    "malformed_tokens": ("malformed_tokens.txt", "0 1\n0 1 2 3\n", {}),
    "malformed_int": ("malformed_int.txt", "0 1\n\n# x\n2 x\n", {}),
    "malformed_float": ("malformed_float.txt", "0 1\n1 2 abc\n", {}),
    "one_token": ("one_token.txt", "0 1\n7\n", {}),
    "mm_pattern": ("mm_pattern.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                   "% a P3\n3 3 2\n2 1\n3 2\n", {}),
    "mm_general": ("mm_general.mtx", "%%MatrixMarket matrix coordinate real general\n"
                   "3 3 1\n1 2 1.0\n", {}),
    "mm_real": ("mm_real.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
                "4 4 3\n2 1 0.5\n3 1 2\n4 4 1.5\n", {"allow_self_loops": True}),
    "mm_isolated": ("mm_isolated.mtx", "%%MatrixMarket matrix coordinate integer symmetric\n"
                    "%c\n\n6 6 2\n2 1\n%mid\n5 3\n", {}),
    "mm_out_of_range": ("mm_oor.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                        "3 3 2\n2 1\n4 2\n", {}),
    "mm_zero_index": ("mm_zero.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                      "3 3 2\n2 1\n0 2\n", {}),
    "mm_count": ("mm_count.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                 "3 3 3\n2 1\n3 2\n", {}),
    "mm_hash_line": ("mm_hash.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                     "3 3 1\n# not a comment here\n2 1\n", {}),
    "mm_bad_header": ("mm_bad_header.mtx", "%%MatrixMarket matrix array real symmetric\n"
                      "3 3\n", {}),
    "mm_no_size": ("mm_no_size.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                   "% only comments\n", {}),
    "mm_not_square": ("mm_not_square.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                      "3 4 1\n2 1\n", {}),
    "mm_sniff_header": ("mm_sniffed.dat", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                        "2 2 1\n2 1\n", {}),
    "empty": ("empty.txt", "", {}),
    "only_comments": ("only_comments.txt", "# a\n% b\n\n   \n", {}),
    "negative_ids": ("negative_ids.txt", "-3 +4\n004 -0\n0\t-3\n", {}),
    "crlf": ("crlf.txt", b"0 1\r\n1 2\r\n# c\r\n2 0", {}),
    "bare_cr": ("bare_cr.txt", b"0 1\r1 2\r2 3\n", {}),
    "underscore": ("underscore.txt", "1_0 2\n2 3\n", {}),
    "int64_overflow": ("overflow.txt", "0 1\n1 99999999999999999999\n", {}),
    "long_ok": ("long_ok.txt", "0 0000000000000000000000001\n1 2\n", {}),
    "both_directions": ("both_dirs.txt", "0 1\n1 0\n1 2\n", {}),
    "same_direction": ("same_dir.txt", "0 1\n0 1\n1 2\n", {}),
    "dir_conflict": ("dir_conflict.txt", "0 1\n0 1\n1 0\n", {}),
    "self_loop": ("self_loop.txt", "0 1\n7 7\n1 2\n", {}),
    "self_loop_ok": ("self_loop_ok.txt", "0 1\n7 7\n1 2\n7 1\n", {"allow_self_loops": True}),
    "self_loop_twice": ("self_loop_twice.txt", "0 1\n1 1\n1 1\n", {"allow_self_loops": True}),
    "weights_all_one": ("w_one.txt", "0 1 1.0\n1 2 1\n", {}),
    "nonpositive_weight": ("w_neg.txt", "0 1 -1.0\n", {}),
    "vt_ff_whitespace": ("vtff.txt", "0\x0b1\n1\x0c2\n", {}),
    "unicode_ws": ("unicode.txt", "0 1\n1 2\n", {}),
    "tab_comment": ("tab_comment.txt", "\t# indented comment\n 0 1\n", {}),
    "fs_whitespace": ("fs_ws.txt", "0\x1c1\n1 2\n", {}),
    "bad_utf8": ("bad_utf8.txt", b"0 1\n\xff 2\n", {}),
    "nul_byte": ("nul.txt", b"0 1\n1\x002\n", {}),
    "random_small": ("random_small.txt", random_edgelist(11, 300, 1000), {}),
    "random_large": ("random_large.txt", random_edgelist(12, 40_000, 60_000), {}),
    "random_weighted": ("random_weighted.txt", random_edgelist(13, 2000, 5000, weighted=True),
                        {}),
    "random_mm": ("random_mm.mtx", random_mm(14, 5000, 30_000), {}),
}


def main():
    os.makedirs(FILES, exist_ok=True)
    out = {}
    for name, (fname, content, kw) in CASES.items():
        path = os.path.join(FILES, fname)
        data = content if isinstance(content, bytes) else content.encode()
        with open(path, "wb") as fh:
            fh.write(data)
        rec = {"file": fname, "kwargs": kw}
        try:
            g, ids = parse_graph_file(path, **kw)
        except Exception as exc:  # noqa: BLE001 -- record the reference's error
            rec["error"] = type(exc).__name__
            rec["message"] = str(exc).replace(path, "{path}")
        else:
            rec.update(n=g.n, nnz=g.nnz, is_weighted=bool(g.is_weighted),
                       num_edges=g.num_edges,
                       row_ptr=sha(g.row_ptr.astype(np.int64)),
                       col_idx=sha(g.col_idx.astype(np.int64)),
                       weights=sha(g.weights.astype(np.float64)),
                       ids=sha(np.asarray(ids, dtype=np.int64)))
            if g.nnz <= 64:
                rec.update(row_ptr_v=g.row_ptr.tolist(), col_idx_v=g.col_idx.tolist(),
                           weights_v=g.weights.tolist(), ids_v=np.asarray(ids).tolist())
        out[name] = rec
        print(name, rec.get("error", ""), rec.get("message", rec.get("n")))
    with open(os.path.join(HERE, "fileio.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
