"""Hot SASS of one kernel from `ncu -i rep --page source --csv --kernel-name regex:K` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iw, ie = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
tot_e = sum(int(r[ie] or 0) for r in data)
tot_w = sum(int(r[iw] or 0) for r in data)
print(f"instructions executed {tot_e}, stall samples {tot_w}, SASS lines {len(data)}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
mode = sys.argv[3] if len(sys.argv) > 3 else "stall"
key = iw if mode == "stall" else ie
for r in sorted(data, key=lambda r: -int(r[key] or 0))[:n]:
    print(f"{r[ia][-5:]} exec={r[ie]:>8s} stall={r[iw]:>6s}  {r[isrc].strip()[:90]}")
