"""Host-side timeline of a solve that takes the robust path (RSVD_B200_TRACE=1 prints a
host timestamp per launch / synchronisation): python tools/probe/robust_trace.py [cfg]."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_03423_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5ill"
cfgd = dict(bench.CONFIGS[name])
if len(sys.argv) > 2:
    cfgd["m"] = cfgd["n"] = int(sys.argv[2])
a = bench.synth_device(torch, cfgd, cfgd["m"], 0, torch.device("cuda", 0))
s = P.Solver(0)
cfg = P.RsvdConfig(k=cfgd["k"], oversample=cfgd["p"], power_q=cfgd["q"], seed=42)
for i in range(int(os.environ.get("SOLVES", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.randomized_ksvd_device(a, cfg)
    torch.cuda.synchronize()
    print(f"solve {i}: {1e3 * (time.perf_counter() - t0):.2f} ms, reruns "
          f"{s.last_info('robust_reruns')}, fallbacks {s.last_info('householder_fallbacks')}",
          file=sys.stderr, flush=True)
