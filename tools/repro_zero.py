import sys, numpy as np
sys.path.insert(0, ".")
import paper_2110_03423_b200 as P
S = P.Solver(0)
a = np.eye(10)
for k in (0, 11):
    try: S.randomized_ksvd(a, P.RsvdConfig(k=k))
    except P.ArgumentError as e: print("ok", e, flush=True)
for bad in (np.nan, np.inf, -np.inf):
    b = np.random.default_rng(0).standard_normal((300, 200)); b[123, 45] = bad
    try: S.randomized_ksvd(b, P.RsvdConfig(k=5))
    except P.ArgumentError as e: print("ok", e, flush=True)
r = S.randomized_ksvd(np.diag([3.0, 2.0, 1.0]), P.RsvdConfig(k=2, seed=3)); print(r.factors.sigma, flush=True)
print("sketch", flush=True)
y = S.sketch(np.zeros((10, 8)), 3, 1); print(np.abs(y).max(), flush=True)
print("fast zero", flush=True)
r = S.randomized_ksvd(np.zeros((30, 20)), P.RsvdConfig(k=3)); print(r.factors.sigma, S.last_info("robust_reruns"), flush=True)
