"""Kernel timeline of repeated graph-replayed solves (torch.profiler / CUPTI): per-kernel device
time, the gaps between consecutive kernels of a solve and the solve's span (probe only).
python tools/probe/gaps.py c1 [reps]"""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
import paper_2110_03423_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = bench.CONFIGS[name]
a = torch.from_numpy(bench.synth_host(cfg)).cuda()
solver = P.Solver()
rc = P.RsvdConfig(k=cfg["k"], oversample=cfg["p"], power_q=cfg["q"], seed=42)
for _ in range(3):
    solver.randomized_ksvd_device(a, rc)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        solver.randomized_ksvd_device(a, rc)
        torch.cuda.synchronize()
path = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
# split into solves at gaps > 200 us
solves, cur = [], [ev[0]]
for e in ev[1:]:
    if e["ts"] - (cur[-1]["ts"] + cur[-1]["dur"]) > 200:
        solves.append(cur)
        cur = []
    cur.append(e)
solves.append(cur)
for s in solves[-3:]:
    busy = sum(e["dur"] for e in s)
    span = s[-1]["ts"] + s[-1]["dur"] - s[0]["ts"]
    gaps = [s[i + 1]["ts"] - (s[i]["ts"] + s[i]["dur"]) for i in range(len(s) - 1)]
    print(f"{len(s)} kernels  span {span:.1f} us  busy {busy:.1f} us  gaps {sum(gaps):.1f} us "
          f"(median {np.median(gaps):.2f}, max {max(gaps):.1f})")
s = solves[-1]
for i, e in enumerate(s):
    g = s[i + 1]["ts"] - (e["ts"] + e["dur"]) if i + 1 < len(s) else 0
    print(f"{e['dur']:8.1f} us  gap {g:6.2f}  {e['name'][:90]}")
