"""A/B check: KPM_BULK=1 (TMA bulk gathers) vs the register-gather path --
moments and T blocks must be bitwise identical."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1905_09758_b200 as kp
from paper_1905_09758_b200 import _lib
from paper_1905_09758_b200.kpm import Run

def run_once(dev, P, mode, steps, bulk, seed=1, hot=None):
    os.environ["KPM_BULK"] = str(bulk)
    if hot: os.environ["KPM_HOT_DEGREE"] = str(hot)
    else: os.environ.pop("KPM_HOT_DEGREE", None)
    M = 2 * steps + 2 if mode == 0 else steps
    run = Run(dev, P, mode, M)
    run.set_probes(kp.make_probes(dev.n, P, "rademacher", seed=seed))
    run.advance(steps)
    ptr, ld, k = run.block()
    blk = np.empty(dev.n * ld)
    _lib.check(_lib.load().kpm_memcpy(_lib.Context.get().handle, _lib.ptr(blk), ctypes.c_void_p(ptr), blk.nbytes, 1))
    _lib.Context.get().synchronize()
    if mode == 2:
        out = np.empty((dev.n, M + 1)); run.result(out, 1.0)
    else:
        out = np.empty((M + 1, run.ld)) if hasattr(run, "ld") else None
        out = None
    run.free()
    return blk, out

ok = True
graphs = {"er": kp.erdos_renyi(3000, 0.01, seed=1).device(), "ba": kp.preferential_attachment(20000, 4, seed=2).device(),
          "rmat16": kp.DeviceGraph.rmat(16, 16, seed=3)}
for name, dev in graphs.items():
    for P in (5, 20, 32, 40, 64, 65, 100, 128):
        for mode in (0, 1, 2):
            a, oa = run_once(dev, P, mode, 5, 0)
            b, ob = run_once(dev, P, mode, 5, 2)
            c, oc = run_once(dev, P, mode, 5, 2, hot=50)
            same = np.array_equal(a, b) and np.array_equal(a, c)
            if oa is not None:
                same = same and np.array_equal(oa, ob) and np.array_equal(oa, oc)
            ok &= same
            print(name, P, mode, "bitwise" if same else "MISMATCH", flush=True)
# moments through the public API
sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(graphs["rmat16"]), (-1.0, 1.0))
z = kp.make_probes(graphs["rmat16"].n, 128, "rademacher", seed=4)
os.environ["KPM_BULK"] = "0"; m0 = kp.dos_moments(sop, z, 60).values
os.environ["KPM_BULK"] = "1"; m1 = kp.dos_moments(sop, z, 60).values
print("moments bitwise", np.array_equal(m0, m1)); ok &= np.array_equal(m0, m1)
print("ALL OK" if ok else "FAILED")
