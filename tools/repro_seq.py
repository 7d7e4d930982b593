"""Replay tests/test_gpu_parity.py in order in one process (bring-up helper)."""
import os, sys, inspect, faulthandler
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import conftest
import test_gpu_parity as T
from oracle.oracle import Oracle
import paper_2110_03423_b200 as P
solver = P.Solver(0)
port = Oracle("port")
import json
meta = json.load(open("tests/golden/cases.json"))
golden = [(c, dict(np.load(f"tests/golden/rsvd_{c['name']}.npz"))) for c in meta["cases"]]
fx = dict(solver=solver, port=port, golden_cases=golden, kat=meta["kat"])
names = [n for n in dir(T) if n.startswith("test_")]
order = sorted(names, key=lambda n: inspect.getsourcelines(getattr(T, n))[1])
stop = sys.argv[1] if len(sys.argv) > 1 else None
for n in order:
    f = getattr(T, n)
    if n == stop:
        os.environ["RSVD_B200_TRACE"] = "1"
    params = inspect.signature(f).parameters
    if n == "test_rsvd_vs_oracle_sizes":
        for args in [(777, 333, 17, 3)]:
            f(solver, port, *args); print("ok", n, args, flush=True)
        continue
    print("run", n, flush=True)
    f(**{k: fx[k] for k in params})
    print("ok", n, flush=True)
