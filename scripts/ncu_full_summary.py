"""Summary of an `ncu --set full` capture for profiles/: per-kernel details (duration, DRAM/compute throughput,
occupancy, issue rate), the warp-stall breakdown from PC sampling, and DRAM bytes per launch.

    python scripts/ncu_full_summary.py <report.ncu-rep> <title>
"""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Compute (SM) Throughput", "L2 Hit Rate", "Theoretical Occupancy", "Issued Warp Per Scheduler",
        "No Eligible", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Executed Ipc Active")


def main():
    rep, title = sys.argv[1], sys.argv[2]
    print(f"# {title}")
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ik, im, iu, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    print("kernel | metric | unit | value")
    for r in rows[1:]:
        if len(r) > iv and r[im] in KEYS:
            print(f"{r[ik][:40]} | {r[im]} | {r[iu]} | {r[iv]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    idx = [i for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")]
    ik = h.index("Kernel Name")
    print("\n# warp stall breakdown (pc sampling, share of samples); dram bytes per launch")
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        vals = sorted(((float(r[i].replace(",", "") or 0), h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                       for i in idx), reverse=True)
        tot = sum(v for v, _ in vals) or 1.0
        rd = r[h.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in h else "?"
        print(r[ik][:40], f"dram_read={rd}{rows[1][h.index('dram__bytes_read.sum')]}" if rd != "?" else "",
              " ".join(f"{n}={v / tot * 100:.0f}%" for v, n in vals[:8]))


if __name__ == "__main__":
    main()
