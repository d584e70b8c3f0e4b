import time, sys, os
sys.path.insert(0, "/root/repo")
import paper_1905_09758_b200 as kp
g = kp.preferential_attachment(1_000_000, 5, seed=1)
tiny = kp.build_csr([(0, 1), (1, 2), (2, 0)])
kp.kpm_pdos(tiny, m_max=4, nz=2, probe_kind="rademacher")
for rep in range(3):
    t = time.perf_counter()
    mom, _ = kp.kpm_pdos(g, m_max=100, nz=64, probe_kind="rademacher", seed=1)
    print("c2 solve", rep, round(time.perf_counter() - t, 4), flush=True)
