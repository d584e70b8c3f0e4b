#!/usr/bin/env python3
"""Benchmark of the KPM hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
                    [--impl ours|reference]

Workload (default ``c5``, BASELINE.json configs[4], the config the north_star's
roofline and scaling targets name): R-MAT scale 26, edge factor 16,
(0.57, 0.19, 0.19, 0.05), seed 4, symmetrised / deduplicated / loop-free
(n = 2^26, nnz = 2.1e9, int32 CSR); global DOS with the 256 Rademacher fp64
probes of ``make_probes(n, 256, seed=4)`` via the doubling recurrence.

Strong scaling: the 256 probe columns are split over the N
ranks (one process per GPU, CSR replicated), each rank runs its columns in
batches of <= 128 (two 68.7 GB recurrence blocks per batch: at N=1 the 256
columns are two sequential batches), and the zero-padded (M+1) x 256
contribution matrix is summed by ONE NCCL all-reduce, inside the timed
region.  A *step* is one fused recurrence step over all 256 probes (each
rank's batches) -- 2 moments per step with doubling; value = nnz * 256 * 2 * K
/ (max over ranks of the device-timed K steps + all-reduce).  Inputs are
resident in HBM; the gathered blocks (34-69 GB per batch) are > 270x the L2.

``e2e`` is the same metric through the public API with host buffers: the host
CSR (int64 row_ptr + int32 col_idx, pinned) is uploaded by rank 0
(``DeviceGraph.from_csr``), replicated to the other ranks by NCCL broadcast
(``distributed.broadcast_graph``), ``dos_moments`` (N=1) or
``distributed.dos_moments_sharded`` (N>1) runs ``--e2e-moments`` moments and
the contributions come back to the host.

``--impl reference`` times the reference's own CPU path on this box's host
cores (rank 0 only): the graph from the oracle's C generator + C restatement
of ``_csr_from_canonical`` (no repo package or GPU code is imported), and the
reference's compiled Cython SpMM (oracle/_ref, built from the reference's
``_spmv.c``) inside the reference's recurrence glue; each timed step is one
recurrence step (one moment, the reference has no doubling) over a bounded
probe sample -- the first W+K moments, SURVEY §8d "first 10 moments".
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    # name: (kind, params, probes, moments)
    "c1": ("er", dict(n=10_000, p=1e-3, seed=0), 20, 200),
    "c2": ("ba", dict(n=1_000_000, m=5, seed=1), 64, 100),
    "c3": ("rmat", dict(scale=24, edge_factor=16, seed=2), 128, 500),
    "c4": ("motif", dict(n_ba=2_000_000, m=4, seed=3), 64, 300),
    "c5": ("rmat", dict(scale=26, edge_factor=16, seed=4), 256, 1000),
    "rmat20": ("rmat", dict(scale=20, edge_factor=16, seed=2), 128, 500),
    "rmat14": ("rmat", dict(scale=14, edge_factor=16, seed=2), 8, 20),  # CPU contract test
}
METRIC = "KPM nnz*probes*moments/sec (G/s) and achieved HBM GB/s"
UNIT = "G nnz*probe*moment/s"
KERNEL_SOURCES = ("paper_1905_09758_b200/csrc/kpm_step.cu",
                  "paper_1905_09758_b200/csrc/kpm_internal.cuh",
                  "paper_1905_09758_b200/csrc/kpm_graph.cu")  # the schedule / twin shape the traffic


def _code_only(src: str) -> str:
    """C++ source without comments and with whitespace collapsed, so that the
    hash follows the code, not its commentary."""
    import re

    src = re.sub(r"/\*.*?\*/", " ", src, flags=re.S)
    src = re.sub(r"//[^\n]*", " ", src)
    return " ".join(src.split())


def kernel_hash() -> str:
    """sha256 of the step kernel's code (comments and whitespace ignored):
    keys profiles/traffic.json (tests/test_bench_contract.py fails when an
    entry there was measured on other code)."""
    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        with open(os.path.join(REPO, f), "r", encoding="utf-8") as fh:
            h.update(_code_only(fh.read()).encode())
    return h.hexdigest()[:16]


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def read_gather_peak():
    """Bandwidth of cold, read-only TMA gather4 traffic on a B200 (GB/s), the
    access pattern of the step kernel, measured by tools/exp/gather_bw.cu
    (profiles/r02_gather_roofline.log) and recorded in profiles/traffic.json.
    MEASURED_PEAKS.json's figure is a COPY (half reads, half writes, with the
    bus turnarounds that costs); a launch that is ~96% reads can exceed it."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            rec = json.load(f)["read_gather_peak"]
        return float(rec["gbs"]), rec["source"]
    except Exception:
        return None, None


def bytes_model(n, nnz, p):
    """SURVEY.md §8d per-nonzero gather model, bytes per fused step over p
    columns: every gathered neighbour row counted (an upper bound on DRAM
    traffic: hot rows are served by L2)."""
    return 4 * nnz + 8 * (n + 1) + 8 * n + 8 * p * nnz + 24 * p * n


def _bytes_per_step(n, nnz, p, ldos=False):
    """bytes_model (+ the LDOS per-node write) for tools/step_timer.py."""
    return bytes_model(n, nnz, p) + (8 * n if ldos else 0)


def bytes_compulsory(n, nnz, p):
    """Every array touched once per step: CSR, d^-1/2, T_k gathered once,
    T_k own rows, T_{k-1} read, T_{k+1} written (a lower bound)."""
    return 4 * nnz + 16 * n + 8 + 8 * p * n + 24 * p * n


def traffic_entry(cfg, p):
    """Measured DRAM bytes of one step launch (ncu dram__bytes_read.sum +
    dram__bytes_write.sum) for this config and batch width, valid only for
    the current kernel sources (profiles/traffic.json, tools/r2/traffic.sh)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            rec = json.load(f)["entries"].get(f"{cfg}/P{p}")
    except Exception:
        return None
    if not rec or rec.get("kernel_sha") != kernel_hash():
        return None
    return rec


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
         "power.draw")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(r[1]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[2]) for r in self.rows) if v is not None]
        pw = [v for v in (num(r[8]) for r in self.rows if len(r) > 8) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(self.rows)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _relaunch(n):
    """--gpus N without torchrun: re-exec this script as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def shard_range(nz, rank, world):
    base, extra = divmod(nz, world)
    c0 = rank * base + min(rank, extra)
    return c0, c0 + base + (1 if rank < extra else 0)


def _workload_name(cfg):
    kind, prm, P, M = CONFIGS[cfg]
    if kind == "rmat":
        return (f"{cfg.upper()}: R-MAT scale {prm['scale']} ef {prm['edge_factor']} "
                f"(0.57,0.19,0.19,0.05) seed {prm['seed']}, global DOS (doubling), "
                f"{P} Rademacher fp64 probes, {M} moments")
    return f"{cfg.upper()}: {kind} {prm}, {P} probes, {M} moments"


# ----------------------------------------------------------------- ours
def build_graph(cfg, ctx):
    import paper_1905_09758_b200 as kp

    kind, prm, _, _ = CONFIGS[cfg]
    if kind == "rmat":
        return kp.DeviceGraph.rmat(prm["scale"], prm["edge_factor"], prm["seed"], ctx=ctx)
    g = host_graph(cfg)
    return kp.DeviceGraph.from_csr(g.n, g.row_ptr, g.col_idx, ctx=ctx)


def host_graph(cfg):
    """Host GraphCSR of an ER / BA / motif-heavy config (the reference's
    generators, restated in paper_1905_09758_b200.testkit, SHA-pinned)."""
    import paper_1905_09758_b200 as kp

    kind, prm, _, _ = CONFIGS[cfg]
    if kind == "er":
        return kp.erdos_renyi(prm["n"], prm["p"], seed=prm["seed"])
    if kind == "ba":
        return kp.preferential_attachment(prm["n"], prm["m"], seed=prm["seed"])
    if kind == "motif":
        return kp.testkit.motif_heavy(prm["n_ba"], prm["m"], prm["seed"])
    raise ValueError(cfg)


def _pinned(a):
    import torch

    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t, t.numpy()


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1905_09758_b200 as kp
    from paper_1905_09758_b200 import _lib
    from paper_1905_09758_b200 import distributed as kdist
    from paper_1905_09758_b200.kpm import Run

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    cuda = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=cuda)
    barrier = (lambda: dist.barrier()) if world > 1 else (lambda: None)
    ctx = _lib.Context.get(local)
    kind, prm, P, M = CONFIGS[args.config]
    seed = prm.get("seed", 0)
    t0 = time.time()
    dev = build_graph(args.config, ctx)
    ctx.synchronize()
    t_build = time.time() - t0
    n, nnz = dev.n, dev.nnz

    twin = dev.prepare(min(P, args.batch))  # builds the gather-ordered twin when runs use it
    c0, c1 = shard_range(P, rank, world)
    emu = args.shard_of if (world == 1 and args.shard_of > 1) else 0
    if emu:  # one GPU runs rank 0's shard of an emu-way split (scaling projection)
        c0, c1 = shard_range(P, 0, emu)
    batches = [(b, min(c1, b + args.batch)) for b in range(c0, c1, args.batch)]
    widths = sorted({b1 - b0 for b0, b1 in batches})
    family = kp.make_probes(n, P, "rademacher", seed=seed)
    K, W = args.steps, args.warmup
    m_run = 2 * (W + K)  # doubling: W + K steps, then the contributions
    contrib = torch.zeros((m_run + 1, P), dtype=torch.float64, device=cuda)
    stream = torch.cuda.ExternalStream(ctx.stream, device=cuda)
    step_ms = kern_ms = 0.0
    launches = 0
    t_probes = 0.0
    with ClockSampler(local) as clk:
        for b0, b1 in batches:
            run = Run(dev, b1 - b0, _lib.MODE_DOS_DOUBLING, m_run)
            try:
                ctx.synchronize()
                tp = time.time()
                run.set_probes(family.column_slice(b0, b1))  # Philox keys -> HBM
                ctx.synchronize()
                t_probes += time.time() - tp
                run.advance(W)
                ctx.synchronize()
                barrier()
                torch.cuda.synchronize()
                run.set_timing(True)
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                run.advance(K)
                ev1.record(stream)
                ev1.synchronize()
                step_ms += ev0.elapsed_time(ev1)
                km, nl = run.kernel_time()
                kern_ms += km
                launches += nl
                part = torch.empty((m_run + 1, b1 - b0), dtype=torch.float64, device=cuda)
                run.result(part.data_ptr())
                contrib[:, b0:b1] = part
            finally:
                run.free()
        # the one collective of the job: sum of the zero-padded contributions
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if world > 1:
            dist.all_reduce(contrib, op=dist.ReduceOp.SUM)
        e1.record()
        e1.synchronize()
        ar_ms = e0.elapsed_time(e1)
    host = contrib.cpu().numpy()
    assert np.isfinite(host).all()
    chk = host[0, c0:c1] if emu else host[0]  # an emulated shard fills its own columns only
    assert np.array_equal(chk, np.full(chk.shape[0], float(n)))  # z_j . z_j = n for +-1 probes

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cuda)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_ms = max_over_ranks(step_ms + ar_ms)
    ms_step = total_ms / K
    kern_avg = max_over_ranks(kern_ms / max(launches, 1))
    units_step = nnz * P * 2
    value = units_step / (ms_step * 1e-3) / 1e9
    if emu:  # this GPU's share only; the projection is reported beside it
        value = nnz * (c1 - c0) * 2 / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel (the fused step over one batch width)
    peak, peak_kind = _peaks()
    pw = max(b1 - b0 for b0, b1 in batches)
    model = bytes_model(n, nnz, pw)
    comp = bytes_compulsory(n, nnz, pw)
    tr = traffic_entry(args.config, pw)
    kern_s = kern_avg * 1e-3
    if tr is not None:
        achieved, basis = tr["dram_bytes"] / kern_s / 1e9, "ncu DRAM bytes per launch"
    else:
        achieved, basis = comp / kern_s / 1e9, "compulsory bytes (no ncu traffic for this kernel hash)"
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4), "traffic": tr["dram_bytes"] if tr else None,
        "basis": basis, "peak_kind": peak_kind,
        "kernel": "kpm_step_g4_kernel (TMA gather4; P>64 as fused 64-column tiles"
                  + ("; gather-ordered twin, evict_first on cold traffic" if twin else "")
                  + f"), batch of {pw} columns",
        "kernel_ms": round(kern_avg, 3), "kernel_sha": kernel_hash(),
        "traffic_source": tr.get("source") if tr else None,
        "frac_model_upper_bound": round(model / kern_s / 1e9 / peak, 4),
        "frac_compulsory_lower_bound": round(comp / kern_s / 1e9 / peak, 4),
        "bytes_per_launch_model": model, "bytes_per_launch_compulsory": comp,
        "frac_nominal_8tbs": round(achieved / 8000.0, 4),
    }
    rpeak, rsrc = read_gather_peak()
    if rpeak:
        roofline["read_peak"] = rpeak
        roofline["frac_of_read_peak"] = round(achieved / rpeak, 4)
        roofline["peak_note"] = (
            "peak is the measured COPY bandwidth (reads + writes); this launch is ~96% reads, "
            "and cold read-only TMA gathers reach read_peak on a B200 (" + rsrc + "), so frac "
            "can pass 1.0 on a box whose clocks hold; traffic is the ncu capture of this kernel "
            "hash, kernel_ms is live")

    want_cpu = rank == 0 and world == 1 and not args.no_cpu
    host_csr = dev.export()[:2] if rank == 0 and (want_cpu or not args.no_e2e) else None
    dev.free()  # the e2e leg uploads its own copy of the graph
    e2e = None
    if not args.no_e2e:
        e2e = _e2e(args, (n, nnz), host_csr, family, world, rank, ctx, barrier, max_over_ranks)

    cpu = None
    if want_cpu:
        # the reference's CPU path on the same CSR (exported from the device;
        # bit-identical to the oracle's, tests/test_gpu_configs.py)
        from oracle import netdos_oracle as orc
        rp, ci = host_csr
        del host_csr
        ci = ci.astype(np.int64)
        cpu = cpu_baseline(args, (rp, ci, orc.normadj_values_c(rp, ci, orc.dinv_of(rp)), 0.0))

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT,
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded R-MAT / Rademacher, no dataset)",
            "config": {"workload": _workload_name(args.config), "n": n, "nnz": nnz,
                       "probes": P, "moments": M, "mode": "doubling (2 moments per step)",
                       "probes_per_gpu": c1 - c0, "batch_widths": widths,
                       "batches_per_gpu": len(batches), "units_per_step": units_step,
                       "parallelism": f"probe-shard x{world} (CSR replicated), one NCCL "
                                      "all-reduce of the (M+1) x P contributions per job",
                       "l2": "inputs larger than L2 (%.1f GB blocks per batch)"
                             % (8 * n * pw / 1e9),
                       "neighbour_order": ("gather-ordered twin: degree-renumbered CSR, rows "
                                           "hottest-first (default at this size; KPM_REORDER=0 "
                                           "= the reference's order)" if twin
                                           else "the reference's CSR order"),
                       "graph_build_s": round(t_build, 3), "probe_gen_s": round(t_probes, 4),
                       "allreduce_ms": round(ar_ms, 3),
                       "per_spmm_value": round(value / 2, 3),
                       "per_spmm_note": "value counts 2 moments per SpMM step (doubling); "
                                        "per_spmm_value counts 1 (the reference's basis)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            # per batch and step: one fused step kernel (all 64-column tiles in
            # one launch) + reduce_groups + finalize
            "gpu_launches": 3 * K * len(batches),
            "clocks": clk.summary(),
        }
        if emu:
            line["emulated_shard"] = {
                "of": emu, "probes": c1 - c0,
                "note": "ONE GPU running rank 0's shard of an %d-way probe split (the per-GPU "
                        "work of the strong-scaling run); value is this GPU's share; "
                        "projected_job_value = %d x value assumes identical shards and the "
                        "measured 2 MB all-reduce hidden (not a multi-GPU measurement)" % (emu, emu),
                "projected_job_value": round(emu * value, 3),
                "projected_ms_per_step": round(ms_step, 4)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _e2e(args, shape, host_csr, family, world, rank, ctx, barrier, max_over_ranks):
    """Same metric through the public API, host buffers in the timed region."""
    import torch

    import paper_1905_09758_b200 as kp
    from paper_1905_09758_b200 import distributed as kdist

    kind, prm, P, M = CONFIGS[args.config]
    n, nnz = shape
    me = args.e2e_moments
    host_rp = host_ci = None
    if rank == 0:
        _t_rp, host_rp = _pinned(host_csr[0])
        _t_ci, host_ci = _pinned(host_csr[1])  # int32: the device layout
    torch.cuda.synchronize()
    barrier()
    t1 = time.perf_counter()
    g = kp.DeviceGraph.from_csr(n, host_rp, host_ci, ctx=ctx) if rank == 0 else None
    g = kdist.broadcast_graph(g, ctx=ctx)
    sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(g), (-1.0, 1.0))
    if world > 1:
        mom = kdist.dos_moments_sharded(sop, family, me)
    else:
        mom = kp.dos_moments(sop, family, me)
    t_e2e = max_over_ranks(time.perf_counter() - t1)
    assert abs(mom.values[0] - 1.0) < 1e-12 and np.isfinite(mom.values).all()
    g.free()
    h2d = (int(host_rp.nbytes + host_ci.nbytes) if host_rp is not None else 0) + 16 * P
    return {"value": round(nnz * P * me / t_e2e / 1e9, 3), "unit": UNIT,
            "seconds": round(t_e2e, 3), "moments": me,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(8 * (me + 1) * P),
            "call": ("DeviceGraph.from_csr(pinned host int64 row_ptr + int32 col_idx) on rank 0"
                     + (" + distributed.broadcast_graph (NCCL) + distributed.dos_moments_sharded"
                        if world > 1 else " + dos_moments") + f"(m_max={me})"),
            "probes": "seeded Rademacher ProbeMatrix regenerated on the device from its "
                      "per-column Philox keys (16 B/column H2D); an explicit host probe block "
                      f"would add {8 * n * P / 1e9:.0f} GB of H2D"}


# ------------------------------------------------------------ CPU side
def _oracle_graph(cfg):
    """The config's CSR on the host in the reference layout (int64 indptr /
    indices, fp64 operator values), built by the oracle only: R-MAT from the
    C generator + C restatement of _csr_from_canonical (bit-identical to the
    device loader, tests/test_gpu_configs.py)."""
    from oracle import netdos_oracle as orc

    kind, prm, P, M = CONFIGS[cfg]
    t0 = time.time()
    if kind == "rmat":
        u, v = orc.rmat_edges(prm["scale"], prm["edge_factor"] << prm["scale"], prm["seed"])
        rp, ci = orc.csr_from_edges(1 << prm["scale"], u, v)
        del u, v
    else:  # ER / BA / motif-heavy: the reference's generators (host numpy)
        g = host_graph(cfg)
        rp, ci = g.row_ptr, g.col_idx
    dinv = orc.dinv_of(rp)
    data = orc.normadj_values_c(rp, ci, dinv)
    return rp, ci, data, time.time() - t0


def _ref_moments(rp, ci, data, z, moments, threads):
    """The reference's recurrence (restated glue, kpm.py:73-108) around its
    compiled Cython csr_matvec: per-moment times after each collect."""
    from oracle import netdos_oracle as orc

    engine = "ref" if orc.ref_spmv() is not None else "c"
    op = orc.CSROp(rp, ci, data, engine=engine)
    stamps = [time.perf_counter()]
    contrib = np.empty((moments + 1, z.shape[1]))

    def collect(m, t):
        contrib[m] = np.einsum("ij,ij->j", z, t)
        stamps.append(time.perf_counter())

    orc.recurrence(op, z, moments, collect, threads)
    return np.diff(np.asarray(stamps))[1:], engine  # moments 1..M


def cpu_baseline(args, graph=None):
    """The reference's CPU path on this host on a bounded sample: moments
    1..2 of `--cpu-probes` columns on all host threads, and moment 1 of one
    column on one thread (SURVEY §8d asks for both)."""
    from oracle import netdos_oracle as orc

    kind, prm, P, M = CONFIGS[args.config]
    rp, ci, data, t_graph = graph or _oracle_graph(args.config)
    n, nnz = rp.shape[0] - 1, ci.shape[0]
    threads = orc.cpu_threads()
    z = np.stack([orc.rademacher_column(n, prm.get("seed", 0), j)
                  for j in range(args.cpu_probes)], 1)
    dt, engine = _ref_moments(rp, ci, data, z, 2, threads)
    dt1, _ = _ref_moments(rp, ci, data, z[:, :1].copy(), 1, 1)
    return {"value": round(nnz * args.cpu_probes / float(np.mean(dt)) / 1e9, 4), "unit": UNIT,
            "cores": threads, "kind": "reference" if engine == "ref" else "port",
            "sample": (f"moments 1-2 (one SpMM + recurrence glue each) of {args.cpu_probes} of "
                       f"{P} probe columns on the full {args.config.upper()} graph (nnz={nnz}); "
                       f"{float(np.mean(dt)):.2f} s per moment; the reference's compiled Cython "
                       "csr_matvec + numpy glue"),
            "single_thread": {"value": round(nnz / float(dt1[0]) / 1e9, 4), "cores": 1,
                              "sample": f"moment 1 of one column; {float(dt1[0]):.2f} s"}}


def run_reference(args):
    """--impl reference: rank 0 alone, host cores only (see module doc)."""
    world, rank, local = _dist_env()
    if rank != 0:
        return
    from oracle import netdos_oracle as orc

    kind, prm, P, M = CONFIGS[args.config]
    rp, ci, data, t_graph = _oracle_graph(args.config)
    n, nnz = rp.shape[0] - 1, ci.shape[0]
    threads = orc.cpu_threads()
    ps = args.ref_probes
    z = np.stack([orc.rademacher_column(n, prm.get("seed", 0), j) for j in range(ps)], 1)
    dt, engine = _ref_moments(rp, ci, data, z, args.warmup + args.steps, threads)
    timed = dt[args.warmup:]
    sec = float(np.mean(timed))
    value = nnz * ps / sec / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded R-MAT / Rademacher, no dataset)",
            "config": {"workload": _workload_name(args.config), "n": n, "nnz": nnz,
                       "probes_sampled": ps, "graph_build_s": round(t_graph, 1),
                       "step": "one recurrence step = one moment (T_{m+1} = 2 H T_m - T_{m-1} "
                               "+ collect), moments W+1..W+K of the sampled columns"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                             "kind": "reference" if engine == "ref" else "port",
                             "sample": f"{args.steps} timed moments (after {args.warmup}) of "
                                       f"{ps} of {P} probe columns; {sec:.2f} s per moment"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=128, help="probe columns per batch")
    ap.add_argument("--e2e-moments", type=int, default=100)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-probes", type=int, default=4)
    ap.add_argument("--ref-probes", type=int, default=2)
    ap.add_argument("--shard-of", type=int, default=0,
                    help="one GPU runs rank 0's shard of an N-way probe split (scaling projection)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args.gpus)
    run_ours(args)


if __name__ == "__main__":
    main()
