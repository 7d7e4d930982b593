"""Locate wrong outputs of the MN-major 3xTF32 GEMM for a given shape."""
import sys, ctypes as C
import torch
sys.path.insert(0, ".")
import paper_2110_03423_b200 as P
S = P.Solver(0)
def run(K, M, NP, splits, out_t=False):
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(K, M, device="cuda", generator=g)
    w = torch.randn(K, NP, device="cuda", generator=g)
    out = torch.full((M, NP), float("nan"), dtype=torch.float64, device="cuda")
    S.wait_for_torch()
    st = S.lib.rsvd_b200_debug_gemm_tf32(S.h, 1, C.c_void_p(a.data_ptr()), M, K, a.stride(0),
        C.c_void_p(w.data_ptr()), w.stride(0), NP, C.c_void_p(out.data_ptr()), out.stride(0), 1, 0, splits)
    assert st == 0, S.lib.rsvd_b200_last_error()
    ref = a.double().T @ w.double()
    bound = a.double().abs().T @ w.double().abs()
    r = ((out - ref).abs() / bound)
    bad = (r > 1e-4) | r.isnan()
    print(f"K={K} M={M} NP={NP} splits={splits}: max {r.max().item():.3e} bad {bad.sum().item()}/{bad.numel()}", end=" ")
    if bad.any():
        rows = bad.any(1).nonzero().flatten(); cols = bad.any(0).nonzero().flatten()
        print(f"rows {rows.min().item()}..{rows.max().item()} ({rows.numel()}) cols {cols.min().item()}..{cols.max().item()} ({cols.numel()})")
    else:
        print()
for K, M, NP, sp in [(20000,1024,272,13),(20000,1024,272,1),(4000,1024,272,13),(20000,1024,256,13),(20000,1024,80,13),(20000,512,272,13),(8000,1024,272,13),(12000,1024,272,13),(16000,1024,272,13)]:
    run(K, M, NP, sp)
