#!/usr/bin/env python3
"""Driver for compute-sanitizer (memcheck / racecheck / synccheck): one small
graph through every light path of the fused step kernel and the other device
kernels, each path checked against the oracle so a run is also a parity run.

    compute-sanitizer --tool racecheck python tools/r2/sanitize_paths.py

Paths (forced with the launch-time env knobs of kpm_step.cu base_params):
gather4 (C=1, C=2), gather4 64-column tiles (fused, P=128; per tile, P=100),
per-lane cp.async "lean" (KPM_G4=0, C<=2), TMA bulk copies (KPM_G4=0
KPM_LEAN=0; also LDOS with P>64), register gathers (KPM_BULK=0 ...), the hub
pipeline (KPM_HEAVY_DEGREE=64), explicit values (Laplacian); plus the
loader, Rademacher, filter, motif scan, LDOS histogram and Lanczos kernels."""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

PATHS = {
    "g4": {},
    "lean": {"KPM_G4": "0"},
    "bulk": {"KPM_G4": "0", "KPM_LEAN": "0"},
    "register": {"KPM_G4": "0", "KPM_LEAN": "0", "KPM_BULK": "0", "KPM_TILE": "0"},
}


def main():
    only = sys.argv[1:]
    hub = os.environ.get("KPM_HEAVY_DEGREE")
    import paper_1905_09758_b200 as kp
    from oracle import netdos_oracle as orc

    g = kp.preferential_attachment(1500, 4, seed=3)
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    data = orc.normadj_values(g.row_ptr, g.col_idx)
    lap = kp.rescale_operator(kp.build_operator(g, "laplacian"), (0.0, 2.0 * g.degrees().max()))
    for name, env in PATHS.items():
        if only and name not in only:
            continue
        for k in ("KPM_G4", "KPM_LEAN", "KPM_BULK", "KPM_TILE"):
            os.environ.pop(k, None)
        os.environ.update(env)
        for P in (20, 50, 100, 128):
            probes = kp.make_probes(g.n, P, "rademacher", seed=1)
            z = probes.columns
            want = orc.c_dos_contrib(g.row_ptr, g.col_idx, data, z, 12)
            got = kp.dos_contrib(sop, probes, 12, doubling=False)
            assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max(), (name, P)
            got2 = kp.dos_contrib(sop, probes, 12)
            assert np.abs(got2 - want).max() <= 1e-9 * np.abs(want).max(), (name, P)
            num = orc.c_ldos_num(g.row_ptr, g.col_idx, data, z, 6)
            pd = kp.pdos_moments(sop, probes, 6)
            assert np.abs(pd.values - (num / num[0]).T).max() <= 1e-12, (name, P)
            lz = kp.dos_contrib(lap, probes, 8, doubling=False)
            b = lap.base
            lw = orc.c_dos_contrib(b.indptr, b.indices, b.data, z, 8, shift=lap.shift,
                                   scale=lap.scale)
            assert np.abs(lz - lw).max() <= 1e-12 * np.abs(lw).max(), (name, P)
            print(f"path {name:9s} P={P:3d} hub={hub}: ok", flush=True)
    if not only:
        # the other device kernels once each
        h = kp.pdos_histogram(sop, kp.make_probes(g.n, 16, "rademacher", seed=2), 20, bins=10,
                              negativity_tol=np.inf)
        assert np.isfinite(h.masses).all()
        res = kp.kpm_dos(g, m_max=20, nz=8, probe_kind="rademacher", seed=3,
                         filter_kinds=("open-twin", "closed-twin", "dangling-two-chain"))
        assert np.isfinite(res.moments.values).all()
        fac = kp.lanczos_factorize(kp.build_operator(g, "laplacian"), np.ones(g.n), 10)
        assert np.isfinite(fac.alphas).all()
        rm = kp.DeviceGraph.rmat(12, 8, 5)
        assert rm.nnz > 0
        print("other kernels: ok", flush=True)


if __name__ == "__main__":
    main()
