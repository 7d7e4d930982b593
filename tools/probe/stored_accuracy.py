import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2110_03423_b200 as P
from oracle.oracle import Oracle
from test_gpu_oz_solves import planted
os.environ["RSVD_B200_GEMM"] = "oz"
port = Oracle("port")
for stored in ("1", "0"):
    os.environ["RSVD_B200_OZ_STORED"] = stored
    solver = P.Solver()
    for (m, n, k, dec, seed, q) in [(3000, 400, 20, 1e12, 13, 3), (4000, 900, 64, 1e4, 4964, 2)]:
        a = planted(m, n, k, dec, seed)
        res = solver.randomized_ksvd(a, P.RsvdConfig(k=k, oversample=10, power_q=q, seed=1))
        ref = port.randomized_ksvd(a, k, oversample=10, power_q=q, seed=1)
        rel = np.abs(res.factors.sigma - ref.sigma) / ref.sigma
        live = ref.sigma > 1e-12 * ref.sigma[0]
        print("stored", stored, (m, n, k, dec), "max rel", rel[live].max(), "fallbacks", solver.last_info("householder_fallbacks"), "at", int(np.argmax(rel)), "sigma ratio", ref.sigma[-1] / ref.sigma[0])
