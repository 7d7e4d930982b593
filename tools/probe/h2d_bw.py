import torch, time
n = 6638764032 // 8
a = torch.empty(n, dtype=torch.float64, pin_memory=True); a.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device='cuda')
for rep in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(a, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"single copy {a.numel()*8/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
# chunked on 2 streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ch = 64 << 20
for rep in range(2):
    torch.cuda.synchronize(); t=time.perf_counter()
    for i, o in enumerate(range(0, n, ch)):
        st = s1 if i % 2 == 0 else s2
        with torch.cuda.stream(st):
            d[o:o+ch].copy_(a[o:o+ch], non_blocking=True)
    torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"2-stream 512MB chunks {a.numel()*8/dt/1e9:.1f} GB/s")
u = torch.empty(202599*64, dtype=torch.float64, pin_memory=True)
du = torch.empty(202599*64, dtype=torch.float64, device='cuda')
torch.cuda.synchronize(); t=time.perf_counter(); u.copy_(du, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
print(f"D2H U {u.numel()*8/dt/1e9:.1f} GB/s ({dt*1e3:.2f} ms)")
import subprocess; print(subprocess.run("nvidia-smi -q | grep -A3 -i 'pcie generation' ; nvidia-smi -q | grep -i 'link width' -A2", shell=True, capture_output=True, text=True).stdout)
