#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, mean, share."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("mpr::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':50s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:50]:50s} {v[0]:8d} {v[1]:10.1f} {v[1] / v[0]:9.2f} {v[1] / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
