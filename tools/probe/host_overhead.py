"""Per-solve host overhead of the device-resident API (probe only): K back-to-back solves timed
with CUDA events (as bench.py does) with and without the NVML clock sampler, against the
device-only span of one solve's graph. python tools/probe/host_overhead.py c1 [K]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2110_03423_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = bench.CONFIGS[name]
a = torch.from_numpy(bench.synth_host(cfg)).cuda()
solver = P.Solver()
rc = P.RsvdConfig(k=cfg["k"], oversample=cfg["p"], power_q=cfg["q"], seed=42)
st = torch.cuda.ExternalStream(solver.stream_handle()) if hasattr(solver, "stream_handle") else None
for _ in range(5):
    solver.randomized_ksvd_device(a, rc)
torch.cuda.synchronize()


def timed(label, sampler=False):
    import contextlib
    ctx = bench.ClockSampler(0) if sampler else contextlib.nullcontext()
    with ctx:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host = 0.0
        for _ in range(K):
            h0 = time.perf_counter()
            solver.randomized_ksvd_device(a, rc)
            host += time.perf_counter() - h0
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    print(f"{label:28s} wall {wall / K * 1e3:.3f} ms/solve  (in the call {host / K * 1e3:.3f})")


timed("no sampler")
timed("with NVML sampler", True)
timed("no sampler")
# host-side cost of the API around the C call
t0 = time.perf_counter()
for _ in range(200):
    sig = torch.empty(64, dtype=torch.float64, device="cuda")
    u = torch.empty((cfg["m"], 64), dtype=torch.float64, device="cuda")
    v = torch.empty((cfg["n"], 64), dtype=torch.float64, device="cuda")
print(f"3 torch.empty: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(200):
    solver.wait_for_torch(a.device)
print(f"wait_for_torch: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
