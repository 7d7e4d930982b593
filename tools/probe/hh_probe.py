"""Time the blocked Householder QR (rsvd_b200_householder_qr_device) on an m x n Gaussian
matrix with graded columns: python tools/probe/hh_probe.py m n [reps]."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_03423_b200 as P  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
s = P.Solver(0)
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
a *= 10.0 ** (-6.0 * torch.arange(n, device="cuda", dtype=torch.float64) / n)
s.householder_qr_device(a)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(s.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(reps):
    s.householder_qr_device(a)
e1.record(st)
e1.synchronize()
print(f"householder_qr {m}x{n}: {e0.elapsed_time(e1) / reps:.3f} ms")
