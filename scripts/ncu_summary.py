"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel medians and the
share of one decode step (library kernels only).  usage: python scripts/ncu_summary.py launches.csv [layers]"""
from __future__ import annotations

import collections
import csv
import statistics
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, ui, vi = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi or "pkv::" not in r[ki]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1000.0 if unit == "ns" else v * 1000.0 if unit == "ms" else v
        out.append((name, us))
    return out


def main():
    path = sys.argv[1]
    rows = load(path)
    by = collections.OrderedDict()
    for name, us in rows:
        by.setdefault(name, []).append(us)
    hot = [k for k in by if k not in ("encode_kernel", "export_kernel", "dbg_scores_kernel", "dbg_cand_kernel")]
    step = sum(statistics.median(by[k]) for k in hot)
    print(f"{'kernel':28s} {'launches':>8s} {'median_us':>10s} {'min_us':>8s} {'share':>6s}")
    for k, v in by.items():
        med = statistics.median(v)
        share = f"{med / step:6.1%}" if k in hot else "   -  "
        print(f"{k:28s} {len(v):8d} {med:10.2f} {min(v):8.2f} {share}")
    print(f"{'sum of hot-path medians (us/layer, serialised, cold)':60s} {step:.2f}")


if __name__ == "__main__":
    main()
