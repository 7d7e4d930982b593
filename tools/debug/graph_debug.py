"""Graph-cache diagnostics: ten device-resident C1 solves with fresh outputs each; run with
RSVD_B200_GRAPH_DEBUG=1 to log every capture."""
import sys, torch
sys.path.insert(0, ".")
import bench, paper_2110_03423_b200 as P
cfgd = bench.CONFIGS["c1"]
dev = torch.device("cuda", 0)
a = bench.synth_device(torch, cfgd, cfgd["m"], 0, dev)
s = P.Solver(0)
cfg = P.RsvdConfig(k=cfgd["k"], oversample=cfgd["p"], power_q=cfgd["q"], seed=42)
# (profiling 0: profiled solves run eagerly)
for i in range(10):
    u, sg, v, sw = s.randomized_ksvd_device(a, cfg)
    print(i, u.data_ptr(), sg.data_ptr(), v.data_ptr(), s.last_info("graph_launches"), file=sys.stderr)
