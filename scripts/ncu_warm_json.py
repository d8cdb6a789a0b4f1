"""profiles/<round>/ncu_warm.json from warm ncu launch lists (gpu__time_duration, no cache flush, serialised):
per configuration the median launch time of each library kernel, and scan_us (read by bench.py for the ncu-timed
scan rate next to the event-timed one).  usage: python scripts/ncu_warm_json.py out.json 128k=a.csv 1m=b.csv"""
from __future__ import annotations

import json
import statistics
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import load  # noqa: E402


def main():
    out = {}
    for arg in sys.argv[2:]:
        cfg, path = arg.split("=", 1)
        per = {}
        for name, us in load(path):
            per.setdefault(name, []).append(us)
        med = {k: round(statistics.median(v), 3) for k, v in per.items()}
        out[cfg] = {"kernels_median_us": med, "launches": {k: len(v) for k, v in per.items()},
                    "scan_us": med.get("scan_kernel"), "source": path.rsplit("/", 1)[-1]}
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
