"""Graph file ingest on the B200.

Mirrors ``netdos.fileio.parse_graph_file`` (fileio.py:104-128): whitespace
edge lists (``u v [w]``, ``#``/``%`` comments; node ids compacted to 0..n-1,
the id map returned alongside the graph) or Matrix Market coordinate
symmetric (1-based, no compaction).  Same return value, same exceptions and
messages (``FileFormatError`` with ``path:lineno``, ``GraphError`` from
``build_csr`` semantics).

Design: the file is read by parallel positional reads into two pinned staging
buffers whose H2D copies overlap the next read; the
device numbers the lines, tokenises one line per thread, compacts the edge
lines, ranks the ids (sort + unique + binary search) and feeds the edges to
the device CSR loader (kpm_graph_from_edges, bit-identical to
``_csr_from_canonical``).  Only the Matrix Market header / size line is read
on the host.

The host parses a file itself only where the device path cannot prove the
reference's result: explicit weights (decimal -> double stays Python's
``float``; ``build_csr`` then sums / checks them), same-direction repeated
edges (weight sums), bytes the device tokenizer does not model (non-ASCII,
bare '\\r', ...), and to word the error of a malformed line.  Those are the
``_host_*`` functions below; they restate fileio.py:28-101 line for line.
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from . import _lib
from .errors import FileFormatError, GraphError
from .graph import DeviceGraph, GraphCSR, build_csr

__all__ = ["parse_graph_file", "load_graph_file", "write_graph_edgelist"]

_INT32_MAX = 0x7FFFFFFF

#: "device" or "host": which path the last parse took (tests / diagnostics)
last_ingest_path = None
#: stage wall times of the last device parse (seconds; tools/ingest_bench.py)
last_ingest_timing: dict = {}


# ------------------------------------------------------------ host restatement
def _host_edgelist_line(path, lineno, s):
    """One non-blank, non-comment edge-list line (fileio.py:34-44)."""
    toks = s.split()
    if len(toks) not in (2, 3):
        raise FileFormatError(f"{path}:{lineno}: expected `u v [w]`, got {s!r}")
    try:
        u, v = int(toks[0]), int(toks[1])
        w = float(toks[2]) if len(toks) == 3 else None
    except ValueError as exc:
        raise FileFormatError(f"{path}:{lineno}: {exc}") from exc
    return (u, v) if w is None else (u, v, w)


def _host_mm_line(path, lineno, s, rows):
    """One Matrix Market entry line (fileio.py:84-94)."""
    toks = s.split()
    if len(toks) not in (2, 3):
        raise FileFormatError(f"{path}:{lineno}: malformed entry {s!r}")
    try:
        i, j = int(toks[0]) - 1, int(toks[1]) - 1
        w = float(toks[2]) if len(toks) == 3 else None
    except ValueError as exc:
        raise FileFormatError(f"{path}:{lineno}: {exc}") from exc
    if not (0 <= i < rows and 0 <= j < rows):
        raise FileFormatError(f"{path}:{lineno}: index out of range")
    return (i, j) if w is None else (i, j, w)


def _host_edgelist(path):
    edges = []
    with open(path) as fh:
        for lineno, line in enumerate(fh, 1):
            s = line.strip()
            if not s or s[0] in "#%":
                continue
            edges.append(_host_edgelist_line(path, lineno, s))
    if not edges:
        raise FileFormatError(f"{path}: no edges found")
    return edges


def _host_matrix_market(path):
    rows, nnz, header_lines, _ = _mm_header(path, check_cr=False)
    edges = []
    with open(path) as fh:
        for _ in range(header_lines):
            fh.readline()
        lineno = header_lines
        for line in fh:
            lineno += 1
            s = line.strip()
            if not s or s.startswith("%"):
                continue
            edges.append(_host_mm_line(path, lineno, s, rows))
    if len(edges) != nnz:
        raise FileFormatError(f"{path}: size line promises {nnz} entries, found {len(edges)}")
    return edges, rows


def _host_compacted(path, edges, allow_self_loops):
    raw = np.array([(e[0], e[1]) for e in edges], dtype=np.int64)
    ids = np.unique(raw)
    lookup = {int(orig): i for i, orig in enumerate(ids.tolist())}
    remapped = [(lookup[e[0]], lookup[e[1]], *e[2:]) for e in edges]
    return build_csr(remapped, n=len(ids), allow_self_loops=allow_self_loops), ids


# ------------------------------------------------------------ Matrix Market head
def _mm_header(path, check_cr=True):
    """Header + size line on the host (fileio.py:50-80).  Returns (rows, nnz,
    number of lines consumed, byte offset of the body)."""
    with open(path) as fh:
        header = fh.readline()
        toks = header.lower().split()
        if len(toks) < 5 or not toks[0].startswith("%%matrixmarket"):
            raise FileFormatError(f"{path}:1: not a MatrixMarket header")
        _, obj, fmt, field, sym = toks[:5]
        if obj != "matrix" or fmt != "coordinate":
            raise FileFormatError(f"{path}:1: only coordinate matrices are supported")
        if field not in ("real", "integer", "pattern"):
            raise FileFormatError(f"{path}:1: unsupported field {field!r}")
        if sym != "symmetric":
            raise FileFormatError(
                f"{path}:1: header declares {sym!r}; undirected graphs need "
                "a symmetric matrix")
        lineno = 1
        size_line = None
        for line in fh:
            lineno += 1
            s = line.strip()
            if not s or s.startswith("%"):
                continue
            size_line = s
            break
    if size_line is None:
        raise FileFormatError(f"{path}: missing size line")
    try:
        rows, cols, nnz = (int(x) for x in size_line.split())
    except ValueError as exc:
        raise FileFormatError(f"{path}:{lineno}: bad size line {size_line!r}") from exc
    if rows != cols:
        raise FileFormatError(f"{path}:{lineno}: matrix must be square, got {rows}x{cols}")
    # byte offset of line `lineno + 1` (the device parses from there); a bare
    # '\r' in the header would make binary and text line numbers disagree
    with open(path, "rb") as fb:
        head = b"".join(fb.readline() for _ in range(lineno))
    if check_cr and head.replace(b"\r\n", b"").count(b"\r"):
        raise _NeedsHost()
    return rows, nnz, lineno, len(head)


# ------------------------------------------------------------ device path
class _DevArrays:
    """Device buffers returned by the ingest entry points (freed on exit)."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.ptrs = []

    def add(self, p):
        if p:
            self.ptrs.append(p)
        return p

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        lib = _lib.load()
        for p in self.ptrs:
            lib.kpm_device_free(self.ctx.handle, ctypes.c_void_p(p))
        self.ptrs.clear()


def _d2h(ctx, dptr, count, dtype):
    out = np.empty(count, dtype=dtype)
    if count:
        _lib.check(_lib.load().kpm_memcpy(ctx.handle, _lib.ptr(out), ctypes.c_void_p(dptr),
                                          out.nbytes, 1), "memcpy")
        ctx.synchronize()
    return out


_STAGE_BYTES = 1 << 27          # 128 MiB per pinned staging buffer
_READ_THREADS = min(8, os.cpu_count() or 1)
_staging = {}


def _pinned_pair(ctx):
    """Two pinned staging buffers per context, allocated once."""
    bufs = _staging.get(ctx.handle)
    if bufs is None:
        lib = _lib.load()
        bufs = []
        for _ in range(2):
            p = ctypes.c_void_p()
            _lib.check(lib.kpm_host_alloc(_STAGE_BYTES, ctypes.byref(p)), "host_alloc")
            bufs.append(p.value)
        _staging[ctx.handle] = bufs
    return bufs


def _read_into(path, offset, addr, nbytes, pool):
    """Parallel positional reads of [offset, offset+nbytes) into host memory
    at addr (page-cache copies release the GIL and scale with threads)."""
    piece = -(-nbytes // _READ_THREADS)

    def one(k):
        lo = k * piece
        hi = min(nbytes, lo + piece)
        if hi <= lo:
            return 0
        view = memoryview((ctypes.c_char * (hi - lo)).from_address(addr + lo)).cast("B")
        with open(path, "rb", buffering=0) as fb:
            fb.seek(offset + lo)
            got = 0
            while got < hi - lo:
                r = fb.readinto(view[got:])
                if not r:
                    break
                got += r
        return got

    got = sum(pool.map(one, range(_READ_THREADS)))
    if got != nbytes:
        raise OSError(f"{path}: short read ({got} of {nbytes} bytes)")


def _upload_file(path, offset, ctx):
    """File bytes [offset, EOF) copied to HBM: parallel reads into two pinned
    staging buffers, each H2D copy overlapping the read of the next chunk.
    Returns (device pointer owned by the caller, size)."""
    from concurrent.futures import ThreadPoolExecutor
    size = max(os.path.getsize(path) - offset, 0)
    if size == 0:
        return None, 0
    lib = _lib.load()
    d = ctypes.c_void_p()
    _lib.check(lib.kpm_device_alloc(ctx.handle, size, ctypes.byref(d)), "device_alloc")
    try:
        stage = _pinned_pair(ctx)
        with ThreadPoolExecutor(_READ_THREADS) as pool:
            pos, k = 0, 0
            while pos < size:
                nb = min(_STAGE_BYTES, size - pos)
                buf = stage[k & 1]
                # buf's previous copy (chunk k-2) was waited for last round;
                # this read overlaps the copy of chunk k-1 from the other buffer
                _read_into(path, offset + pos, buf, nb, pool)
                ctx.synchronize()
                _lib.check(lib.kpm_memcpy(ctx.handle, ctypes.c_void_p(d.value + pos),
                                          ctypes.c_void_p(buf), nb, 0), "memcpy")
                pos += nb
                k += 1
        ctx.synchronize()
    except BaseException:
        lib.kpm_device_free(ctx.handle, d)
        raise
    return d.value, size


def _line_text(path, lineno):
    with open(path) as fh:
        for k, line in enumerate(fh, 1):
            if k == lineno:
                return line.strip()
    return ""


class _NeedsHost(Exception):
    pass


def _device_ingest(path, mm, allow_self_loops, ctx):
    """Returns (DeviceGraph, ids or None) or raises _NeedsHost / the
    reference's errors."""
    lib = _lib.load()
    if mm is not None:
        rows, nnz, header_lines, offset = mm
        base, flags = 1, 0
    else:
        header_lines, offset, base, flags = 0, 0, 0, _lib.KPM_PARSE_HASH_COMMENTS
    t0 = time.perf_counter()
    dtext, size = _upload_file(path, offset, ctx)
    t1 = time.perf_counter()
    last_ingest_timing.clear()
    last_ingest_timing.update(bytes=size, upload_s=t1 - t0)
    with _DevArrays(ctx) as bufs:
        nl = ctypes.c_int64()
        du, dv, ds = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        unusual = ctypes.c_int32()
        try:
            rc = lib.kpm_parse_edges(ctx.handle, ctypes.c_void_p(dtext), size, base, flags,
                                     ctypes.byref(nl), ctypes.byref(du), ctypes.byref(dv),
                                     ctypes.byref(ds), ctypes.byref(unusual))
        finally:
            if dtext:
                lib.kpm_device_free(ctx.handle, ctypes.c_void_p(dtext))
        _lib.check(rc, "parse_edges")
        for p in (du.value, dv.value, ds.value):
            bufs.add(p)
        if unusual.value:
            raise _NeedsHost()
        nlines = nl.value
        t2 = time.perf_counter()
        last_ingest_timing.update(parse_s=t2 - t1, lines=nlines)
        m, n = ctypes.c_int64(), ctypes.c_int64()
        eu, ev, dids = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        info = (ctypes.c_int32 * 5)()
        _lib.check(lib.kpm_edges_finalize(
            ctx.handle, nlines, du, dv, ds, 0 if mm is not None else 1,
            rows if mm is not None else 0, ctypes.byref(m), ctypes.byref(n), ctypes.byref(eu),
            ctypes.byref(ev), ctypes.byref(dids), info), "edges_finalize")
        for p in (eu.value, ev.value, dids.value):
            bufs.add(p)
        t3 = time.perf_counter()
        last_ingest_timing.update(finalize_s=t3 - t2)
        if info[0] & 2:
            raise _NeedsHost()  # ids Python's int() must judge ('_', > 18 digits)
        if info[3] != _INT32_MAX or (mm is not None and info[4]):
            # first offending line in file order (malformed, or MM index
            # out of range); the host words the reference's error for it
            first = info[3] if info[3] != _INT32_MAX else nlines
            if mm is not None and info[4]:
                status = _d2h(ctx, ds.value, nlines, np.int8)
                u = _d2h(ctx, du.value, nlines, np.int64)
                v = _d2h(ctx, dv.value, nlines, np.int64)
                kept = status >= 2
                oor = kept & ((u < 0) | (u >= rows) | (v < 0) | (v >= rows))
                if oor.any():
                    first = min(first, int(np.argmax(oor)))
            lineno = header_lines + first + 1
            s = _line_text(path, lineno)
            if mm is not None:
                _host_mm_line(path, lineno, s, rows)
            else:
                _host_edgelist_line(path, lineno, s)
            raise AssertionError(f"{path}:{lineno}: device flagged a line the host accepts")
        if info[0] or info[2]:
            raise _NeedsHost()  # weights / weight sums: build_csr semantics on the host
        m, n = m.value, n.value
        if mm is not None:
            if m != nnz:
                raise FileFormatError(
                    f"{path}: size line promises {nnz} entries, found {m}")
        elif m == 0:
            raise FileFormatError(f"{path}: no edges found")
        if info[1] and not allow_self_loops:
            u = _d2h(ctx, eu.value, m, np.int64)
            v = _d2h(ctx, ev.value, m, np.int64)
            node = int(u[np.argmax(u == v)])
            raise GraphError(f"self-loop at node {node} (pass allow_self_loops to accept)")
        ids = _d2h(ctx, dids.value, n, np.int64) if mm is None else np.arange(n, dtype=np.int64)
        h = ctypes.c_void_p()
        _lib.check(lib.kpm_graph_from_edges(ctx.handle, n, eu, ev, m,
                                            1 if allow_self_loops else 0, ctypes.byref(h)),
                   "graph_from_edges")
        last_ingest_timing.update(load_s=time.perf_counter() - t3, edges=m)
        return DeviceGraph(h.value, ctx), ids


def _sniff(path, fmt):
    if fmt is None:
        fmt = "matrix_market" if str(path).endswith((".mtx", ".mm")) else None
        if fmt is None:
            with open(path) as fh:
                first = fh.readline()
            fmt = "matrix_market" if first.lower().startswith("%%matrixmarket") else "edgelist"
    if fmt not in ("matrix_market", "edgelist"):
        raise ValueError(f"unknown graph format {fmt!r}")
    return fmt


def _ingest(path, fmt, allow_self_loops, ctx):
    """(DeviceGraph | None, GraphCSR | None, ids): the device graph when the
    device path holds, else the host-built GraphCSR."""
    fmt = _sniff(path, fmt)
    ctx = ctx or _lib.Context.get()
    global last_ingest_path
    last_ingest_path = "device"   # also when the device path raises the error
    try:
        mm = _mm_header(path) if fmt == "matrix_market" else None
        dev, ids = _device_ingest(path, mm, allow_self_loops, ctx)
        return dev, None, ids
    except _NeedsHost:
        pass
    last_ingest_path = "host"
    g, ids = _host_parse(path, fmt, allow_self_loops)
    return None, g, ids


def _host_parse(path, fmt, allow_self_loops):
    """The host restatement of parse_graph_file (fileio.py:104-128) for the
    files the device path hands back (see the module docstring)."""
    fmt = _sniff(path, fmt)
    if fmt == "matrix_market":
        edges, rows = _host_matrix_market(path)
        return build_csr(edges, n=rows, allow_self_loops=allow_self_loops), \
            np.arange(rows, dtype=np.int64)
    return _host_compacted(path, _host_edgelist(path), allow_self_loops)


def parse_graph_file(path, fmt=None, allow_self_loops=False, ctx=None):
    """Drop-in for ``netdos.parse_graph_file`` (fileio.py:104-128): returns
    (GraphCSR, node_id_map); node_id_map[i] is the original id of node i."""
    dev, g, ids = _ingest(path, fmt, allow_self_loops, ctx)
    if dev is not None:
        g = dev.to_host()
        dev.free()
    return g, ids


def load_graph_file(path, fmt=None, allow_self_loops=False, ctx=None):
    """Same parse, graph left in HBM: (DeviceGraph, node_id_map).  A
    DeviceGraph is the unit-weight graph whose normalized adjacency the
    kernels form from degrees, so a file whose parsed weights are not all 1
    -- explicit weights, or a same-direction repeated edge, which build_csr
    sums to weight 2 (graph.py:145-155) -- raises GraphError; such files go
    through parse_graph_file + build_operator (explicit values)."""
    dev, g, ids = _ingest(path, fmt, allow_self_loops, ctx)
    if dev is None:
        if not g.unit_weights:
            raise GraphError("load_graph_file: the parsed graph has non-unit edge weights "
                             "(explicit weights or repeated edges), which have no implicit "
                             "normalized-adjacency device form; use parse_graph_file")
        dev = DeviceGraph.from_csr(g.n, g.row_ptr, g.col_idx, ctx=ctx)
    return dev, ids


def write_graph_edgelist(g: GraphCSR, path, node_ids=None):
    """Canonical ``u v [w]`` lines (fileio.py:131-142)."""
    u, v, w = g.edge_list()
    if node_ids is not None:
        u, v = np.asarray(node_ids)[u], np.asarray(node_ids)[v]
    with open(path, "w") as fh:
        fh.write(f"# nodes {g.n} edges {u.shape[0]}\n")
        if g.is_weighted:
            fh.writelines(f"{a} {b} {ww!r}\n" for a, b, ww in zip(u.tolist(), v.tolist(),
                                                                   w.tolist()))
        else:
            fh.writelines(f"{a} {b}\n" for a, b in zip(u.tolist(), v.tolist()))
