"""Summarise an `ncu --csv --log-file` launch list: per kernel name, launches,
mean duration (us), mean DRAM bytes (read+write) and their share of the total.

    python scripts/ncu_summary.py gpurun_out/launches.csv [--md]
"""
import csv
import re
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"])
            v = d["Metric Value"].replace(",", "")
            try:
                recs.setdefault(key, {})[d["Metric Name"]] = float(v)
            except ValueError:
                pass
    return recs


def short(name):
    m = re.search(r"(\w+_kernel|\w+Kernel|\w+)\s*[<(]", name)
    return m.group(1) if m else name[:50]


def summarize(path):
    recs = load(path)
    agg = OrderedDict()
    for (i, name), m in sorted(recs.items()):
        a = agg.setdefault(short(name), {"n": 0, "t": 0.0, "bytes": 0.0})
        a["n"] += 1
        a["t"] += m.get("gpu__time_duration.sum", 0.0)
        a["bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["t"] for a in agg.values()) or 1.0
    return agg, tot


if __name__ == "__main__":
    agg, tot = summarize(sys.argv[1])
    md = "--md" in sys.argv
    if md:
        print("| kernel | launches | mean us | share of time | mean DRAM MB/launch | GB/s |")
        print("|---|---|---|---|---|---|")
    for k, a in agg.items():
        mt = a["t"] / a["n"] / 1e3
        mb = a["bytes"] / a["n"] / 1e6
        gbs = a["bytes"] / a["t"] if a["t"] else 0.0
        if md:
            print(f"| {k} | {a['n']} | {mt:.1f} | {a['t']/tot:.1%} | {mb:.1f} | {gbs:.0f} |")
        else:
            print(f"{k:40s} n={a['n']:4d} mean={mt:9.1f}us share={a['t']/tot:6.1%} dram={mb:9.1f}MB {gbs:7.0f}GB/s")
