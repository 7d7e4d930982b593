"""Time the K-major 3xTF32 GEMM (debug C-ABI, synchronous) at C4's M x K for several NP."""
import ctypes as C
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2110_03423_b200 as P  # noqa: E402

s = P.Solver(0)
M, K = 200000, 4096
a = torch.randn(M, K, device="cuda", dtype=torch.float32)
for NP in [int(x) for x in sys.argv[1:]] or [256, 272]:
    b = torch.randn(NP, K, device="cuda", dtype=torch.float32)
    out = torch.empty(M, NP, device="cuda", dtype=torch.float32)
    s.wait_for_torch()
    def call():
        st = s.lib.rsvd_b200_debug_gemm_tf32(s.h, 0, C.c_void_p(a.data_ptr()), M, K, K,
                                            C.c_void_p(b.data_ptr()), K, NP,
                                            C.c_void_p(out.data_ptr()), NP, 0, 0, 1)
        assert st == 0
    call()
    t = time.perf_counter()
    for _ in range(10):
        call()
    dt = (time.perf_counter() - t) / 10
    print(f"NP={NP}: {dt*1e3:.3f} ms  {2*M*K*NP/dt/1e12:.1f} TF algorithmic", flush=True)
