import os, sys, threading
import numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2110_03423_b200 as P
from test_gpu_sharded import planted
os.environ["RSVD_B200_UPLOAD_CHUNK_MB"] = sys.argv[1] if len(sys.argv) > 1 else "1"
m, n = 8192, 512
a = planted(m, n, lambda i: np.exp(-i / 15.0), 12)
cfg = P.RsvdConfig(k=32, power_q=int(sys.argv[3]) if len(sys.argv) > 3 else 2, seed=7)
for world in (1, 2) if len(sys.argv) < 3 else (int(sys.argv[2]),):
    group = P.LocalGroup(world)
    solvers = [P.Solver(0) for _ in range(world)]
    for r, s in enumerate(solvers): s.attach_local(group, r)
    spans = [P.shard_rows(m, world, r) for r in range(world)]
    res = [None]*world
    def work(r):
        r0, r1 = spans[r]; s = solvers[r]; shard = np.ascontiguousarray(a[r0:r1])
        h = s.randomized_ksvd_sharded(shard, m, cfg); sp = s.last_info("upload_aty_splits")
        u, sg, v, _ = s.randomized_ksvd_sharded_device(torch.from_numpy(shard).cuda(), m, cfg)
        torch.cuda.synchronize()
        res[r] = (h, sp, sg.cpu().numpy())
    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [t.start() for t in th]; [t.join() for t in th]
    for s in solvers: s.detach()
    for r in range(world):
        h, sp, sg = res[r]
        print(world, r, "splits", sp, "max sigma diff", np.abs(h.factors.sigma - sg).max())
