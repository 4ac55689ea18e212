"""Per-SASS-instruction execution counts and stall samples of one kernel in an ncu report.

    python scripts/sass_hot.py report.ncu-rep [min_samples]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))[1:]
h, rows = r[0], r[1:]
ie, sm = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot_i = sum(int(x[ie] or 0) for x in rows)
tot_s = sum(int(x[sm] or 0) for x in rows)
print(f"instructions {tot_i}  samples {tot_s}")
for i, x in enumerate(rows):
    if int(x[sm] or 0) >= lim:
        print(f"{i:5d} {int(x[ie] or 0):9d} {x[sm]:>5s}  {x[1][:90]}")
