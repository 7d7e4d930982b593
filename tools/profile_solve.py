"""One warm-up + one profiled C2 solve (device-resident A), for ncu launch lists.
The kernels of the second solve are the last `launches` entries of the ncu log."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_03423_b200 as P  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else bench.M
n = int(sys.argv[2]) if len(sys.argv) > 2 else bench.N
dev = torch.device("cuda", 0)
a = bench.synth_device(torch, m, n, 42, dev)
s = P.Solver(0)
cfg = P.RsvdConfig(k=bench.K_RANK, oversample=bench.P_OVER, power_q=bench.Q_POW, seed=42)
torch.cuda.synchronize()
for _ in range(2):
    s.randomized_ksvd_device(a, cfg)
torch.cuda.synchronize()
print("launches per solve", s.last_launch_count())
