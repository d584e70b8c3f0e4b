import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1905_09758_b200 as kp
from paper_1905_09758_b200 import motifs as M
kp._lib.Context.get().synchronize()
g = kp.testkit.motif_heavy()
t=time.time(); insts = kp.detect_motifs(g, seed=3); print("detect", time.time()-t)
p = kp.make_probes(g.n, 64, "rademacher", seed=3)
t=time.time(); cols = p.columns; print("host probe columns", time.time()-t)
t=time.time(); fast = M._deflation_from_arrays(insts.arrays, g.n); print("deflation arrays", time.time()-t)
t=time.time(); out = M._project_csr(cols, fast[0]); print("project (H2D+kernel+D2H)", time.time()-t)
sop = kp.scaled_operator_for(g, "normalized-adjacency")
pf = kp.with_columns(p, out)
t=time.time(); m = kp.dos_moments(sop, pf, 300, effective_dim=g.n - 757575); print("dos_moments (first: graph upload)", time.time()-t)
t=time.time(); m = kp.dos_moments(sop, pf, 300, effective_dim=g.n - 757575); print("dos_moments (warm)", time.time()-t)
