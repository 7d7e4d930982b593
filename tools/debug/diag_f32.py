"""FP32 (3xTF32) path accuracy at C4 size vs the planted spectrum and vs the FP64 path."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2110_03423_b200 as P
S = P.Solver(0)
m, n, k, r = 200000, 4096, 256, 264
g = torch.Generator(device="cuda").manual_seed(7)
u = torch.linalg.qr(torch.randn(m, r, dtype=torch.float64, device="cuda", generator=g))[0]
v = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g))[0]
sig = torch.exp(-torch.arange(r, dtype=torch.float64, device="cuda") / 120.0)
a = ((u * sig) @ v.T).float()
a64 = a.double()
for q in (4, 0, 1):
    cfg = P.RsvdConfig(k=k, oversample=16, power_q=q, seed=42)
    uf, sf, vf, _ = S.randomized_ksvd_f32_device(a, cfg)
    ud, sd, vd, _ = S.randomized_ksvd_device(a64, cfg)
    relf = ((sf - sig[:k]).abs() / sig[:k]); reld = ((sd - sig[:k]).abs() / sig[:k])
    rel32 = ((sf - sd).abs() / sd)
    print(f"q={q}: f32 vs planted max {relf.max().item():.2e} at {relf.argmax().item()} (first {relf[0].item():.2e} median {relf.median().item():.2e}); "
          f"f64 vs planted {reld.max().item():.2e}; f32 vs f64 {rel32.max().item():.2e}; "
          f"orth U {((uf.T@uf)-torch.eye(k,device='cuda',dtype=torch.float64)).abs().max().item():.1e}", flush=True)
