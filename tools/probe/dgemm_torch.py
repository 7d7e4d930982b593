import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for (m, n, k) in [(8192, 8192, 8192), (202599, 80, 4096), (4096, 80, 202599)]:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"torch/cuBLAS DGEMM {m}x{n}x{k}: {best:.3f} ms  {2*m*n*k/best/1e9:.2f} TFLOP/s")
# AtX shape: (k x m)^T
a = torch.randn(202599, 4096, dtype=torch.float64, device="cuda"); w = torch.randn(202599, 80, dtype=torch.float64, device="cuda")
for _ in range(3): z = a.t() @ w
torch.cuda.synchronize(); e0.record(); z = a.t() @ w; e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)
print(f"cuBLAS A^T W 202599x4096 s=80: {ms:.3f} ms {2*202599*4096*80/ms/1e9:.2f} TFLOP/s")
