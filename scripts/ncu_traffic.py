"""profiles/ncu_traffic.json from an `ncu --page raw --csv` export of a `--set full` capture:
dram__bytes_read.sum + dram__bytes_write.sum per launch, keyed by bench.py's kernel names.

    python scripts/ncu_traffic.py <raw.csv> <config> [profiles/ncu_traffic.json]
"""
import csv
import json
import os
import statistics
import sys

NAMES = {"qprep_kernel": "qprep", "scan_kernel": "scan", "select_kernel": "select", "rerank_cpt_kernel": "rerank",
         "rerank_kernel": "rerank", "rerank_flat_kernel": "rerank", "topk_cl_kernel": "topk", "topk_kernel": "topk", "merge_kernel": "topk_merge",
         "attend_partial_kernel": "attend"}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    src, config = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "profiles", "r02",
                                                              "ncu_traffic.json")
    rows = list(csv.reader(open(src)))
    hdr = rows[0]
    units = rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        kname = r[col["Kernel Name"]]
        key = next((v for k, v in NAMES.items() if k in kname), None)
        if key is None:
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[col[m]].replace(",", "")) * SCALE[units[col[m]]]
        per.setdefault(key, []).append(b)
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[config] = {k: round(statistics.median(v)) for k, v in per.items()}
    data["_source"] = ("ncu --set full --clock-control none (L2 flushed before each kernel): "
                       "dram__bytes_read.sum + dram__bytes_write.sum per launch, median over captured launches")
    json.dump(data, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[config]))


if __name__ == "__main__":
    main()
