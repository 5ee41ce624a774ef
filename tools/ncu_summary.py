"""Summarise an ncu --csv launch list: per-kernel launches, time share, DRAM bytes.

    python tools/ncu_summary.py gpurun_out/launches_c2.csv > profiles/xxx.md
"""

from __future__ import annotations

import csv
import re
import sys
from collections import defaultdict


def load(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    out = defaultdict(dict)  # launch id -> {name, metric: value}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        lid = r[ix["ID"]]
        out[lid]["name"] = r[ix["Kernel Name"]]
        unit = r[ix["Metric Unit"]]
        val = float(r[ix["Metric Value"]].replace(",", "")) if r[ix["Metric Value"]] else 0.0
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        out[lid][r[ix["Metric Name"]]] = val * scale
    return out


def short(name):
    m = re.match(r"(?:void )?(?:uqg::)?([A-Za-z_0-9]+)", name)
    base = m.group(1) if m else name
    t = re.search(r"<([^>]*)>", name)
    return base + (f"<{t.group(1)}>" if t else "")


def main(path):
    launches = load(path)
    agg = defaultdict(lambda: {"n": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
    for rec in launches.values():
        a = agg[short(rec["name"])]
        a["n"] += 1
        a["us"] += rec.get("gpu__time_duration.sum", 0.0)
        a["rd"] += rec.get("dram__bytes_read.sum", 0.0)
        a["wr"] += rec.get("dram__bytes_write.sum", 0.0)
    total = sum(a["us"] for a in agg.values()) or 1.0
    print(f"source: {path}  ({len(launches)} launches, serialised, cold-cache per launch)\n")
    print("| kernel | launches | total ms | share | avg us | DRAM read+write per launch (MB) | GB/s |")
    print("|---|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        per = (a["rd"] + a["wr"]) / max(a["n"], 1) / 1e6
        gbs = (a["rd"] + a["wr"]) / (a["us"] * 1e-6) / 1e9 if a["us"] else 0.0
        print(f"| {k} | {a['n']} | {a['us'] / 1e3:.2f} | {100 * a['us'] / total:.1f}% | "
              f"{a['us'] / max(a['n'], 1):.1f} | {per:.2f} | {gbs:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1])
