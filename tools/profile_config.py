"""Two device-resident solves of a bench config (the second is the one to read in an ncu
launch list): python tools/profile_config.py [c1|c2|c3|c4|c5]."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_03423_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfgd = bench.CONFIGS[name]
dev = torch.device("cuda", 0)
a = bench.synth_device(torch, cfgd, cfgd["m"], 0, dev)
if cfgd.get("f32"):
    a = a.float()
s = P.Solver(0)
cfg = P.RsvdConfig(k=cfgd["k"], oversample=cfgd["p"], power_q=cfgd["q"], seed=42)
solve = s.randomized_ksvd_f32_device if cfgd.get("f32") else s.randomized_ksvd_device
torch.cuda.synchronize()
for _ in range(2):
    solve(a, cfg)
torch.cuda.synchronize()
print("launches per solve", s.last_launch_count())
