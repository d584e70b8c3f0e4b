"""Race / ordering stress of the asynchronous pipelines (mbarrier rings, TMA
gather4 and bulk copies into shared memory, cp.async rings, the atomic work
queue).  compute-sanitizer is closed on the GPU pool
(profiles/r02_sanitizer_unavailable.log), so the evidence is behavioural: on a
graph large enough to keep every SM's 16 warps busy (R-MAT scale 16, 1.6e6
nonzeros, forced hub rows), every light path is run repeatedly and each run's
T block must be BITWISE equal to the oracle's sequential recurrence -- a
missing wait, a slot reused early or a torn row shows up as a differing bit.
"""

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from paper_1905_09758_b200 import _lib
from paper_1905_09758_b200.kpm import Run

pytestmark = pytest.mark.gpu

_PATHS = {
    "tiles": {},
    "tiles-unfused": {"KPM_FUSE_TILES": "0"},
    "g4": {"KPM_G4": "2", "KPM_TILE": "0"},
    "lean": {"KPM_G4": "0"},
    "bulk": {"KPM_G4": "0", "KPM_LEAN": "0"},
    "register": {"KPM_G4": "0", "KPM_LEAN": "0", "KPM_BULK": "0"},
}
_KEYS = ("KPM_G4", "KPM_TILE", "KPM_LEAN", "KPM_BULK", "KPM_HEAVY_DEGREE", "KPM_G4_HOT",
         "KPM_HOT_MB_G4", "KPM_FUSE_TILES")


def _block(dev, probes, mode, steps, ctx):
    run = Run(dev, probes.nz, mode, 2 * steps + 2)
    try:
        run.set_probes(probes)
        run.advance(steps)
        ptr, ld, _ = run.block()
        out = np.empty((dev.n, ld))
        _lib.check(_lib.load().kpm_memcpy(ctx.handle, _lib.ptr(out), ptr, out.nbytes, 1))
        ctx.synchronize()
        return out[:, :probes.nz].copy()
    finally:
        run.free()


@pytest.fixture(scope="module")
def rmat16(oracle):
    scale, ef, seed = 16, 12, 9
    u, v = oracle.rmat_edges(scale, ef << scale, seed)
    rp, ci = oracle.csr_from_edges(1 << scale, u, v)
    data = oracle.normadj_values(rp, ci, oracle.dinv_of(rp))
    return scale, ef, seed, rp, ci, data


@pytest.mark.parametrize("P", [32, 64, 128])
def test_twin_runs_repeat_bitwise(oracle, kpm_ctx, monkeypatch, rmat16, P):
    """The gather-ordered twin (KPM_REORDER=1, a hot set small enough that
    gather4 groups mix hinted and unhinted copies): repeated runs are bitwise
    equal to each other and within rounding of the oracle."""
    scale, ef, seed, rp, ci, data = rmat16
    for k in _KEYS:
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("KPM_REORDER", "1")
    monkeypatch.setenv("KPM_HOT_ROWS", "500")
    monkeypatch.setenv("KPM_HEAVY_DEGREE", "3000")
    dev = kp.DeviceGraph.rmat(scale, ef, seed)
    probes = kp.make_probes(dev.n, P, "rademacher", seed=P)
    want = oracle.c_recurrence_block(rp, ci, data, probes.columns, 4, threads=8)
    for mode in (_lib.MODE_DOS_DOUBLING, _lib.MODE_LDOS):
        first = _block(dev, probes, mode, 4, kpm_ctx)
        assert np.max(np.abs(first - want)) <= 1e-13 * np.max(np.abs(want))
        for rep in range(5):
            assert np.array_equal(_block(dev, probes, mode, 4, kpm_ctx), first), (P, mode, rep)
    dev.free()


@pytest.mark.parametrize("path", sorted(_PATHS))
@pytest.mark.parametrize("P", [32, 64, 128])
def test_repeated_runs_bitwise_equal_oracle(oracle, kpm_ctx, monkeypatch, rmat16, path, P):
    scale, ef, seed, rp, ci, data = rmat16
    for k in _KEYS:
        monkeypatch.delenv(k, raising=False)
    for k, v in _PATHS[path].items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("KPM_HEAVY_DEGREE", "3000")  # a few dozen hub rows
    dev = kp.DeviceGraph.rmat(scale, ef, seed)
    assert dev.nnz == ci.shape[0]
    probes = kp.make_probes(dev.n, P, "rademacher", seed=P)
    z = probes.columns
    steps = 4
    want = oracle.c_recurrence_block(rp, ci, data, z, steps, threads=8)
    for mode in (_lib.MODE_DOS_DOUBLING, _lib.MODE_LDOS):
        for rep in range(6):
            got = _block(dev, probes, mode, steps, kpm_ctx)
            assert np.array_equal(got, want), (path, P, mode, rep)
    dev.free()
