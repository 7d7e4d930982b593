"""Summarise an ncu launch list (gpu__time_duration.sum) for the last solve of a run:
python tools/launch_summary.py launches.csv [marker-kernel-substring]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
marker = sys.argv[2] if len(sys.argv) > 2 else "omega"
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]; data = rows[i + 1:]
ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); gi = hdr.index("Grid Size")
ours = data  # every launch of the run is the library's (profile_config.py)
idx = [j for j, r in enumerate(ours) if marker in r[ki]]
last = ours[idx[-1]:] if idx else ours
agg = defaultdict(float); cnt = defaultdict(int); tot = 0
for r in last:
    ms = float(r[vi]) / 1e6
    name = r[ki].split("(")[0].replace("void ", "")[:70]
    agg[name] += ms; cnt[name] += 1; tot += ms
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:70s} {cnt[k]:4d} {v:8.3f} ms {v / tot * 100:5.1f}%")
print(f"total {tot:.3f} ms over {len(last)} launches")
