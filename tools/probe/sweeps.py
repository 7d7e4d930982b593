"""Jacobi sweeps of the pipeline's small SVD per bench config (probe)."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_03423_b200 as P  # noqa: E402

for name in sys.argv[1:]:
    cfgd = bench.CONFIGS[name]
    a = bench.synth_device(torch, cfgd, cfgd["m"], 0, torch.device("cuda", 0))
    if cfgd.get("f32"):
        a = a.float()
    s = P.Solver(0)
    cfg = P.RsvdConfig(k=cfgd["k"], oversample=cfgd["p"], power_q=cfgd["q"], seed=42)
    (s.randomized_ksvd_f32_device if cfgd.get("f32") else s.randomized_ksvd_device)(a, cfg)
    torch.cuda.synchronize()
    print(name, "jacobi sweeps", s.last_info("jacobi_sweeps"), flush=True)
    del a
    torch.cuda.empty_cache()
