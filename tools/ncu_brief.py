"""Brief of an ncu --set full report: duration, pipes, stall mix, top stalled SASS lines.
python tools/ncu_brief.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
want = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__warps_active.avg.per_cycle_active"]
for w in want:
    if w in h:
        print(f"{w:70s} {v[h.index(w)]}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
sh, rows = src[1], src[2:]
si = sh.index("Warp Stall Sampling (All Samples)")
ex = sh.index("Instructions Executed")
cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: 0 for c in cols}
for x in rows:
    for c in cols:
        try:
            tot[c] += int(x[sh.index(c)])
        except (ValueError, IndexError):
            pass
s = sum(tot.values()) or 1
print("stall mix:", ", ".join(f"{c[6:]} {100 * n / s:.1f}%" for c, n in sorted(tot.items(), key=lambda t: -t[1])[:8]))
def num(x, i):
    try:
        return int(x[i] or 0)
    except (ValueError, IndexError):
        return 0


for x in sorted(rows, key=lambda x: -num(x, si))[:ntop]:
    st = sorted(((c[6:], num(x, sh.index(c))) for c in cols), key=lambda t: -t[1])[:2]
    print(f"{x[0][-5:]} {x[1][:56]:56s} {x[si]:>7s} exec {x[ex]:>9s} {st}")
