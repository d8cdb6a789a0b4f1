"""Compare selected raw ncu metrics of one kernel across captures: python scripts/ncu_cmp.py <regex> a_raw.csv b_raw.csv ..."""
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    return h, units, data[0] if data else None


def main():
    pat = re.compile(sys.argv[1])
    caps = [load(p) for p in sys.argv[2:]]
    h0 = caps[0][0]
    names = [n for n in h0 if pat.search(n)]
    print("metric".ljust(70), " | ".join(p.split("/")[-1][:18].ljust(18) for p in sys.argv[2:]))
    for n in names:
        vals = []
        for h, u, r in caps:
            vals.append((r[h.index(n)] if r is not None and n in h else "-") + " " + (u[h.index(n)] if n in h else ""))
        print(n[:70].ljust(70), " | ".join(v[:18].ljust(18) for v in vals))


if __name__ == "__main__":
    main()
