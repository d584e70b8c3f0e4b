#!/usr/bin/env python3
"""Benchmark of the KPM hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
                    [--impl ours|reference]

Workload (default ``c3``, BASELINE.json configs[2]): R-MAT scale 24, edge factor
16, (0.57, 0.19, 0.19, 0.05), seed 2, symmetrised / deduplicated / loop-free,
int32 CSR; global DOS with 128 Rademacher fp64 probes and 500 Chebyshev moments
via the doubling recurrence.  It is the largest BASELINE config that runs on one
GPU in one pass (C5 needs 275 GB of recurrence blocks for its 256 probes, i.e.
two sequential probe batches on one B200).

A *step* is one fused recurrence step (SpMM + three-term update + moment
reduction, plus the deterministic finalize) over the whole probe block; with
doubling each step yields 2 moments, so units/step = nnz * P * 2.  Inputs are
resident in HBM (17.2 GB per block >> 126 MB L2, so no L2 flush is needed).

Multi-GPU (torchrun, one process per GPU): weak scaling -- every rank runs the
same graph with its own 128-column range of a 128*N-column probe family
(probe sharding, no data-path collective); value = all ranks' units / max time.

``--impl reference`` times the reference's own CPU path on this box's host
cores: its compiled Cython SpMM (oracle/_ref, built from the reference's
_spmv.c) inside the reference's recurrence glue (restated with the identical
numpy calls), on the same config and metric, one recurrence step over a
bounded probe sample per timed step.
"""

from __future__ import annotations

import argparse
import json
import os
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
}
METRIC = "KPM nnz*probes*moments/sec (G/s) and achieved HBM GB/s"


def _tiled(P):
    """kpm_step.cu launch_c: P > 64 probes (4-column layout, ld % 4 == 0) run
    as 64-column TMA gather4 passes unless KPM_TILE=0 / KPM_G4=0."""
    ld = -(-P // 4) * 4
    return (P > 64 and ld % 4 == 0 and os.environ.get("KPM_TILE", "1") != "0"
            and os.environ.get("KPM_G4", "1") != "0")


def _step_launches(P):
    # the 64-column tiles of one step run as one launch when ld % 64 == 0
    # (KPM_FUSE_TILES, kpm_step.cu launch_c), else one launch per tile
    ld = -(-P // 4) * 4
    if not _tiled(P):
        return 1
    return 1 if ld % 64 == 0 and os.environ.get("KPM_FUSE_TILES", "1") != "0" else -(-P // 64)


def _kernel_label(P):
    if _tiled(P):
        return ("kpm_step_g4_kernel<C=2,DBL>, %d 64-column tiles in %d launch(es) (TMA gather4)"
                % (-(-P // 64), _step_launches(P)))
    if P <= 64 and os.environ.get("KPM_G4", "1") != "0":
        return "kpm_step_g4_kernel<DBL> (TMA gather4)"
    if os.environ.get("KPM_BULK", "2") != "0":
        return "kpm_step_bulk_kernel<DBL> (TMA bulk-copy gathers)"
    return "kpm_step_kernel<DBL>"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _bytes_per_step(n, nnz, p, ldos=False):
    """SURVEY.md §8d per-nonzero gather model (bytes per fused step launch)."""
    b = 4 * nnz + 8 * (n + 1) + 8 * n + 8 * p * nnz + 24 * p * n
    return b + (8 * n if ldos else 0)


def _compulsory_bytes(n, nnz, p):
    return 4 * nnz + 16 * n + 8 + 8 * p * n + 24 * p * n


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

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
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _init_dist(world, local):
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def _barrier(dist):
    if dist is not None:
        dist.barrier()


def _max_over_ranks(dist, x):
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def build_graph(cfg, ctx):
    import paper_1905_09758_b200 as kp

    kind, prm, _, _ = CONFIGS[cfg]
    if kind == "rmat":
        return kp.DeviceGraph.rmat(prm["scale"], prm["edge_factor"], prm["seed"], ctx=ctx)
    g = host_graph(cfg)
    return kp.DeviceGraph.from_csr(g.n, g.row_ptr, g.col_idx, ctx=ctx)


def host_graph(cfg):
    """Host GraphCSR of an ER / BA / motif-heavy config (reference generators)."""
    import paper_1905_09758_b200 as kp

    kind, prm, _, _ = CONFIGS[cfg]
    if kind == "er":
        return kp.erdos_renyi(prm["n"], prm["p"], seed=prm["seed"])
    if kind == "ba":
        return kp.preferential_attachment(prm["n"], prm["m"], seed=prm["seed"])
    if kind == "motif":
        return kp.testkit.motif_heavy(prm["n_ba"], prm["m"], prm["seed"])
    raise ValueError(cfg)


# ----------------------------------------------------------------- ours
def run_ours(args):
    import torch

    import paper_1905_09758_b200 as kp
    from paper_1905_09758_b200 import _lib
    from paper_1905_09758_b200.kpm import Run

    world, rank, local = _dist_env()
    dist = _init_dist(world, local)
    ctx = _lib.Context.get(local)
    kind, prm, P, M = CONFIGS[args.config]
    t0 = time.time()
    dev = build_graph(args.config, ctx)
    t_build = time.time() - t0
    n, nnz = dev.n, dev.nnz

    steps_needed = args.warmup + args.steps
    m_run = max(M, 2 * steps_needed)
    family = kp.make_probes(n, P * world, "rademacher", seed=prm.get("seed", 0))
    probes = family.column_slice(rank * P, (rank + 1) * P)
    run = Run(dev, P, _lib.MODE_DOS_DOUBLING, m_run)
    ctx.synchronize()
    t0 = time.time()
    run.set_probes(probes)  # seeded Rademacher columns generated in HBM
    ctx.synchronize()
    t_probes = time.time() - t0
    stream = torch.cuda.ExternalStream(ctx.stream, device=local)
    torch.cuda.set_device(local)

    run.advance(args.warmup)
    ctx.synchronize()
    _barrier(dist)
    torch.cuda.synchronize()
    run.set_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        run.advance(args.steps)
        ev1.record(stream)
        ctx.synchronize()
        torch.cuda.synchronize()
    _barrier(dist)
    elapsed = ev0.elapsed_time(ev1)  # ms
    kern_ms, launches = run.kernel_time()
    run.free()
    ms_step = _max_over_ranks(dist, elapsed / args.steps)
    kern_avg = _max_over_ranks(dist, kern_ms / max(launches, 1))
    units_step = nnz * P * 2 * world
    value = units_step / (ms_step * 1e-3) / 1e9

    peak, peak_kind = _peaks()
    bstep = _bytes_per_step(n, nnz, P)
    achieved = bstep / (kern_avg * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.config)
        except Exception:
            traffic = None

    # ---- e2e through the public API with host buffers (rank 0 timing, all
    # ranks run it): host CSR (pinned) -> device graph -> probes from host keys
    # -> full M-moment dos_moments -> contrib D2H -> host moments.
    e2e = None
    if not args.no_e2e:
        rp, ci, _ = dev.export()
        host_rp = _pinned_copy(rp)
        host_ci = _pinned_copy(ci.astype(np.int64))
        del rp, ci
        dev.free()
        _barrier(dist)
        t1 = time.perf_counter()
        g2 = kp.DeviceGraph.from_csr(n, host_rp, host_ci, ctx=ctx)
        op = kp.NormalizedAdjacencyOperator(g2)
        sop = kp.rescale_operator(op, (-1.0, 1.0))
        mom = kp.dos_moments(sop, probes, M)
        t_e2e = time.perf_counter() - t1
        t_e2e = _max_over_ranks(dist, t_e2e)
        assert np.isfinite(mom.values).all() and abs(mom.values[0] - 1.0) < 1e-12
        e2e = {"value": nnz * P * M * world / t_e2e / 1e9, "unit": "G nnz*probe*moment/s",
               "seconds": round(t_e2e, 4),
               "h2d_bytes_per_step": int(host_rp.nbytes + host_ci.nbytes + 16 * P),
               "d2h_bytes_per_step": int(8 * (M + 1) * P),
               "call": "DeviceGraph.from_csr(host int64 CSR) + dos_moments(M=%d)" % M}
        g2.free()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, sample_probes=args.cpu_probes, sample_steps=1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "G nnz*probe*moment/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_name(args.config), "n": n, "nnz": nnz,
                       "probes_per_gpu": P, "moments": M, "mode": "doubling",
                       "units_per_step": units_step, "parallelism": f"probe-shard x{world}",
                       "l2": "inputs larger than L2 (two %.1f GB blocks)" % (8 * n * P / 1e9),
                       "graph_build_s": round(t_build, 3), "probe_gen_s": round(t_probes, 4)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "frac_nominal_8tbs": round(achieved / 8000.0, 4),
                         "bytes_per_launch_model": bstep,
                         "bytes_per_launch_compulsory": _compulsory_bytes(n, nnz, P),
                         "kernel": _kernel_label(P),
                         "kernel_ms": round(kern_avg, 4),
                         "hbm_gbs_model_per_step": round(bstep / (ms_step * 1e-3) / 1e9, 1),
                         # measured DRAM bytes per step (ncu, profiles/traffic.json; all tile launches)
                         # over the live kernel time: the DRAM-side fraction
                         "traffic_GBs": (round(traffic / (kern_avg * 1e-3) / 1e9, 1)
                                         if traffic else None),
                         "traffic_frac": (round(traffic / (kern_avg * 1e-3) / 1e9 / peak, 4)
                                          if traffic else None)},
            "cpu_baseline": cpu, "e2e": e2e,
            # per step: the step kernel (one launch per 64-column tile) +
            # reduce_groups + finalize
            "gpu_launches": (_step_launches(P) + 2) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _pinned_copy(a):
    import torch

    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def _workload_name(cfg):
    kind, prm, P, M = CONFIGS[cfg]
    if kind == "rmat":
        return (f"{cfg.upper()}: R-MAT scale {prm['scale']} ef {prm['edge_factor']} "
                f"seed {prm['seed']}, global DOS, {P} Rademacher probes, {M} moments")
    return f"{cfg.upper()}: ER n={prm['n']} p={prm['p']} seed {prm['seed']}, {P} probes, {M} moments"


# ------------------------------------------------------------ CPU baseline
def _host_graph(cfg):
    """The config's CSR on the host in the reference layout (int64 indptr /
    indices, fp64 h values), built with the device loader when a GPU is
    present (input preparation, outside every timed region), else with the
    oracle's C generator + CSR builder."""
    from oracle import netdos_oracle as orc

    kind, prm, P, M = CONFIGS[cfg]
    try:
        import paper_1905_09758_b200 as kp
        from paper_1905_09758_b200 import _lib

        ctx = _lib.Context.get(int(os.environ.get("LOCAL_RANK", "0")))
        dev = build_graph(cfg, ctx)
        rp, ci, dinv = dev.export()
        dev.free()
        ci = ci.astype(np.int64)
    except Exception:
        if kind == "rmat":
            u, v = orc.rmat_edges(prm["scale"], prm["edge_factor"] << prm["scale"], prm["seed"])
            rp, ci = orc.csr_from_edges(1 << prm["scale"], u, v)
        else:
            from paper_1905_09758_b200.testkit import erdos_renyi
            g = erdos_renyi(prm["n"], prm["p"], seed=prm["seed"])
            rp, ci = g.row_ptr, g.col_idx
        dinv = orc.dinv_of(rp)
    data = orc.normadj_values(rp, ci, dinv)
    return rp, ci, data


def cpu_baseline(cfg, sample_probes=8, sample_steps=1, graph=None):
    """The reference's CPU path (its compiled Cython kernel + the recurrence
    glue) on a bounded sample: `sample_steps` recurrence steps over the first
    `sample_probes` probe columns, all host threads."""
    from oracle import netdos_oracle as orc

    kind, prm, P, M = CONFIGS[cfg]
    rp, ci, data = graph if graph is not None else _host_graph(cfg)
    n = rp.shape[0] - 1
    nnz = ci.shape[0]
    threads = orc.cpu_threads()
    engine = "ref" if orc.ref_spmv() is not None else "c"
    z = orc.make_probes(n, sample_probes, "rademacher", seed=prm.get("seed", 0))
    op = orc.CSROp(rp, ci, data, engine=engine)
    t0 = time.perf_counter()
    orc.dos_contrib(op, z, sample_steps, threads=threads)
    dt = time.perf_counter() - t0
    # SURVEY §8d also asks for threads=1 (the numpy glue is single-threaded,
    # so cores scale poorly): 2 probe columns, one step
    z1 = z[:, :2].copy()
    t0 = time.perf_counter()
    orc.dos_contrib(op, z1, sample_steps, threads=1)
    dt1 = time.perf_counter() - t0
    return {"value": round(nnz * sample_probes * sample_steps / dt / 1e9, 4),
            "unit": "G nnz*probe*moment/s", "cores": threads,
            "kind": "reference" if engine == "ref" else "port",
            "sample": (f"{sample_steps} recurrence step(s) (dos_moments m_max={sample_steps}) "
                       f"over {sample_probes} of {P} probes on the full {cfg.upper()} graph "
                       f"(nnz={nnz}); {dt:.2f} s; reference Cython csr_matvec + numpy glue"),
            "single_thread": {"value": round(nnz * 2 * sample_steps / dt1 / 1e9, 4),
                              "cores": 1,
                              "sample": f"{sample_steps} step(s) over 2 probe columns; {dt1:.2f} s"}}


def run_reference(args):
    world, rank, local = _dist_env()
    if rank != 0:
        return
    from oracle import netdos_oracle as orc

    kind, prm, P, M = CONFIGS[args.config]
    graph = _host_graph(args.config)
    rp, ci, data = graph
    n, nnz = rp.shape[0] - 1, ci.shape[0]
    threads = orc.cpu_threads()
    engine = "ref" if orc.ref_spmv() is not None else "c"
    op = orc.CSROp(rp, ci, data, engine=engine)
    ps = args.cpu_probes
    z = orc.make_probes(n, ps, "rademacher", seed=prm.get("seed", 0))
    for _ in range(args.warmup):
        orc.dos_contrib(op, z, 1, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.dos_contrib(op, z, 1, threads=threads)
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    value = nnz * ps / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4),
            "unit": "G nnz*probe*moment/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_name(args.config), "n": n, "nnz": nnz,
                       "probes_sampled": ps},
            "cpu_baseline": {"value": round(value, 4), "unit": "G nnz*probe*moment/s",
                             "cores": threads, "kind": "reference" if engine == "ref" else "port",
                             "sample": f"one recurrence step (T_1 = H z + collect) over {ps} "
                                       f"probe columns per timed step"},
            "e2e": {"value": round(value, 4), "unit": "G nnz*probe*moment/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-probes", type=int, default=8)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
