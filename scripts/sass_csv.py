"""Summarise an exported ncu SASS source page (scripts/prof_src.sh): total warp instructions,
the executed count of every instruction, grouped into runs of equal count (basic blocks).

    python scripts/sass_csv.py gpurun_out/src/sbs_scan_sass.csv [units] [min_share]
"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
lim = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
h, data = rows[1], rows[2:]
ie, sm, ad, sr = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Address"), h.index("Source")
tot = sum(int(r[ie] or 0) for r in data)
tots = sum(int(r[sm] or 0) for r in data)
print(f"warp instructions {tot}  per unit {tot / units:.1f}  stall samples {tots}")
blocks, cur = [], None
for r in data:
    c = int(r[ie] or 0)
    if cur and cur[1] == c:
        cur[2] += 1; cur[3] += int(r[sm] or 0); cur[4].append(r[sr])
    else:
        cur = [r[ad], c, 1, int(r[sm] or 0), [r[sr]]]; blocks.append(cur)
for a, c, n, s, src in blocks:
    share = c * n / tot * 100
    if share >= lim:
        print(f"{a:>8} exec {c:9d} x {n:3d} instr = {share:5.1f}%  per unit {c * n / units:6.2f}  stalls {s:6d}  first: {src[0][:60]}")
