"""Time the INT8-emulated FP64 GEMM (rsvd_b200_debug_gemm_oz) at a pass-over-A shape: the ax
pass Y = A X (m x n by n x NP) and the atx pass Z^T = (A^T W)^T, each run twice (read the
second in an ncu launch list). python tools/probe/oz_time.py [m n NP cols splits]"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2110_03423_b200 as P  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
m, n, NP, cols, splits = (int(x) for x in (args[:5] if len(args) > 4 else
                                            (202599, 4096, 80, 74, 23)))
s = P.Solver(0)
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
xt = torch.zeros(NP, n, dtype=torch.float64, device="cuda")
xt[:cols] = torch.randn(cols, n, dtype=torch.float64, device="cuda", generator=g)
w = torch.zeros(m, NP, dtype=torch.float64, device="cuda")
w[:, :cols] = torch.randn(m, cols, dtype=torch.float64, device="cuda", generator=g)
y = torch.empty(m, NP, dtype=torch.float64, device="cuda")
zt = torch.empty(NP, n, dtype=torch.float64, device="cuda")
z = torch.empty(n, NP, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
hook = getattr(s.lib, "rsvd_b200_debug_gemm_ozd" if "--stored" in sys.argv else "rsvd_b200_debug_gemm_oz")
for rep in range(2):
    t0 = time.perf_counter()
    st = hook(s.h, 0, C.c_void_p(a.data_ptr()), m, n, n,
                                       C.c_void_p(xt.data_ptr()), n, NP, cols,
                                       C.c_void_p(y.data_ptr()), NP, 0, 1)
    assert st == 0, s.lib.rsvd_b200_last_error().decode()
    t1 = time.perf_counter()
    if "--stored" in sys.argv:  # the stored-digit atx writes Z (n x NP), not Z^T
        st = hook(s.h, 1, C.c_void_p(a.data_ptr()), n, m, n, C.c_void_p(w.data_ptr()), NP, NP,
                  cols, C.c_void_p(z.data_ptr()), NP, 0, splits)
    else:
        st = hook(s.h, 1, C.c_void_p(a.data_ptr()), n, m, n,
                                       C.c_void_p(w.data_ptr()), NP, NP, cols,
                                       C.c_void_p(zt.data_ptr()), n, 1, splits)
    assert st == 0, s.lib.rsvd_b200_last_error().decode()
    t2 = time.perf_counter()
    print(f"rep {rep}: ax call {1e3 * (t1 - t0):.2f} ms, atx call {1e3 * (t2 - t1):.2f} ms (wall, incl. scan+digits)")
ref = (a[:1000] @ xt.T)
print("ax max rel err (first 1000 rows):", ((y[:1000] - ref).abs().max() / ref.abs().max()).item())
ref2 = (a.T @ w).T
zz = z.T if "--stored" in sys.argv else zt
print("atx max rel err:", ((zz - ref2).abs().max() / ref2.abs().max()).item())
