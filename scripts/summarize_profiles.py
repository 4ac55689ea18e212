"""Summarise a per-round profile (scripts/profile_round.sh output) into profiles/:

    python scripts/summarize_profiles.py gpurun_out/prof r01

writes profiles/<round>_launches_cfg3.csv (the raw launch list),
profiles/<round>_ncu_summary.md (per-kernel share + --set full headline
metrics, stall mix, hottest SASS lines) and updates profiles/ncu_traffic.json
(DRAM bytes per launch of each kernel from the --set full captures; bench.py
reads the gather-attend entry as roofline.traffic).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = ["sbs_sample_mma_kernel", "sbs_scan_kernel", "sbs_select_kernel", "attend_union_ws_kernel",
           "merge_parts_kernel"]
WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Waves Per SM", "L2 Hit Rate"]


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full_summary(rep, n_hot=8):
    rows = page(rep, "--page", "details")
    h = rows[0]
    head = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in WANT and d["Metric Name"] not in head:
            head[d["Metric Name"]] = f"{d['Metric Value']} {d.get('Metric Unit', '')}".strip()
    raw = page(rep, "--page", "raw")
    d = dict(zip(raw[0], raw[2]))
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((k[33:], float(v)))
            except ValueError:
                pass
    tot = sum(v for _, v in st) or 1.0
    stalls = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st, key=lambda t: -t[1])[:6])
    num = lambda k: float(str(d.get(k, "0")).replace(",", "") or 0)
    dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    # raw dram__bytes are reported in the unit of row 1 (usually Mbyte)
    unit = dict(zip(raw[0], raw[1])).get("dram__bytes_read.sum", "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    src = page(rep, "--page", "source", "--print-source", "sass")
    hot = []
    if len(src) > 2:
        hh = src[1]
        ie, sc, ss = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
        data = [r for r in src[2:] if len(r) > ss]
        for r in sorted(data, key=lambda r: -float(r[ss] or 0))[:n_hot]:
            hot.append(f"`{r[sc].strip()[:60]}` (samples {r[ss]})")
    return head, stalls, dram * scale, num("smsp__inst_executed.sum"), hot


def main():
    src_dir, rnd = sys.argv[1], sys.argv[2]
    prof = os.environ.get("PROFILES_DIR", os.path.join(ROOT, "profiles"))
    os.makedirs(prof, exist_ok=True)
    shutil.copy(os.path.join(src_dir, "launches.csv"), os.path.join(prof, f"{rnd}_launches_cfg3.csv"))
    agg, tot = ncu_summary.summarize(os.path.join(src_dir, "launches.csv"))
    lines = [f"# {rnd}: ncu profile of the fused step at cfg3 (B=16, N=131072, S=50, bf16)", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dense --no-graph` "
             f"(raw: `{rnd}_launches_cfg3.csv`). Durations are serialised and cold-ish (ncu replays); "
             "the kernel SHARE is what bench.py's live `phases_us` must agree with.", "",
             "| kernel | launches | mean us | share | DRAM MB/launch | GB/s |", "|---|---|---|---|---|---|"]
    fused = {k: v for k, v in agg.items() if k in KERNELS}
    ftot = sum(a["t"] for a in fused.values()) or 1.0
    for k, a in fused.items():
        n = a["n"]
        lines.append(f"| {k} | {n} | {a['t'] / n / 1e3:.1f} | {a['t'] / ftot:.1%} | {a['bytes'] / n / 1e6:.1f} | "
                     f"{a['bytes'] / a['t']:.0f} |")
    traffic = {}
    for k in KERNELS:
        rep = os.path.join(src_dir, f"{k}.ncu-rep")
        if not os.path.exists(rep):
            continue
        head, stalls, dram, inst, hot = full_summary(rep)
        traffic[k] = dram
        lines += ["", f"## {k} (`ncu --set full`, one launch)", ""]
        lines += [f"- {m}: {v}" for m, v in head.items()]
        lines += [f"- DRAM bytes (read + write): {dram / 1e6:.1f} MB; instructions: {inst / 1e6:.1f} M",
                  f"- stall mix: {stalls}", "- hottest SASS lines: " + "; ".join(hot)]
    open(os.path.join(prof, f"{rnd}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    tp = os.path.join(prof, "ncu_traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    ent = tj.setdefault("cfg3", {})
    ent["kernels"] = traffic
    ent["round"] = rnd
    ent["dram_bytes_per_step"] = sum(traffic.values())
    json.dump(tj, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
