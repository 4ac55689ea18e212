mkdir -p gpurun_out/sp
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sbs_scan_kernel -s 3 -c 1 -o gpurun_out/sp/scan \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dense --no-graph > gpurun_out/sp/scan.log 2>&1
python scripts/ncu_lines.py gpurun_out/sp/scan.ncu-rep 60 > gpurun_out/sp/lines.txt 2>&1
python - > gpurun_out/sp/lines_by_inst.txt 2>&1 <<'PY'
import subprocess, csv, io
rep = "gpurun_out/sp/scan.ncu-rep"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]; si = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
agg = {}; cur = None; fname = None
for r in rows[hi + 1:]:
    if not r: continue
    if r[0] in ("File Path", "File Name"): fname = r[1].split("/")[-1]; continue
    if r[0]: cur = (fname, int(r[0]), r[1].strip()[:90]); agg.setdefault(cur, [0.0, 0.0])
    if cur and len(r) > ei and r[2]:
        try: agg[cur][0] += float(r[si] or 0); agg[cur][1] += float(r[ei] or 0)
        except ValueError: pass
te = sum(v[1] for v in agg.values())
print("total warp instructions", te)
for k, v in sorted(agg.items(), key=lambda kv: (str(kv[0][0]), kv[0][1])):
    if v[1] > 0.002 * te:
        print(f"{100*v[1]/te:5.1f}% inst {100*v[0]/max(1,sum(x[0] for x in agg.values())):5.1f}% samp  {k[0]}:{k[1]} {k[2]}")
PY
rm -f gpurun_out/sp/scan.ncu-rep
