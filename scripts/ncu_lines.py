"""Stall samples and executed instructions per CUDA source line of one kernel
in an ncu report (mixed cuda+sass source page).

    python scripts/ncu_lines.py report.ncu-rep [n]
"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
agg = {}
cur = None
fname = None
for r in rows[hi + 1:]:
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:90])
        agg.setdefault(cur, [0.0, 0.0])
    if cur and len(r) > ei and r[2]:
        try:
            agg[cur][0] += float(r[si] or 0)
            agg[cur][1] += float(r[ei] or 0)
        except ValueError:
            pass
tot_s = sum(v[0] for v in agg.values()) or 1
tot_e = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s:.0f}, warp instructions {tot_e:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * v[0] / tot_s:5.1f}% samp {100 * v[1] / tot_e:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
