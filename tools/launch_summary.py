"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: launches,
total device time and share of the captured step(s).  ncu serialises and cold-starts every launch,
so compare SHARES with bench.py's per-op CUDA-event breakdown, not absolutes.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    n = 0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        us = v * scale
        name = re.sub(r"\(.*", "", r[ki]).replace("sarathi::", "").replace("<unnamed>::", "").strip()
        agg[name][0] += 1
        agg[name][1] += us
        total += us
        n += 1
    print(f"# ncu launch list {sys.argv[1]}: {n} launches, {total:.1f} us total (serialised, cold)")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {c:8d} {t:10.1f} {t / c:8.2f} {100 * t / total:5.1f}%")


if __name__ == "__main__":
    main()
