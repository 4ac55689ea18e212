"""Summarise one kernel of an ncu --set full report: headline metrics, stall mix, hottest SASS lines.

    python scripts/ncu_brief.py report.ncu-rep [n_hot]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n_hot = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("--page", "details")
h = rows[0]
want = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "DRAM Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Block Limit Registers", "Block Limit Shared Mem", "Waves Per SM",
        "L2 Hit Rate", "Memory Throughput"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:32s} {d['Metric Value']} {d.get('Metric Unit', '')}")
raw = page("--page", "raw")
d = dict(zip(raw[0], raw[2]))
st = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((k[33:], float(v)))
        except ValueError:
            pass
tot = sum(v for _, v in st) or 1
print("stalls:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(st, key=lambda t: -t[1])[:8]))
for k in ["smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]:
    print(k, d.get(k))
src = page("--page", "source", "--print-source", "sass")
hh = src[1]
ie, sc, ss = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
data = [r for r in src[2:] if len(r) > ss]
print(f"{len(data)} SASS lines; hottest by stall samples:")
for r in sorted(data, key=lambda r: -float(r[ss] or 0))[:n_hot]:
    print(f"  {r[0][-5:]} {r[sc].strip()[:70]:70s} exec={r[ie]} samples={r[ss]}")
