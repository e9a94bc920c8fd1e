"""Print the headline ncu metrics (and top stall reasons) of every kernel in a report.

    python scripts/ncu_kernels.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Grid Size", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Static Shared Memory Per Block", "Dynamic Shared Memory Per Block"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ik, iid, im, iv, iu = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    cur = None
    for r in rows[1:]:
        if (r[iid], r[ik]) != cur:
            cur = (r[iid], r[ik])
            print(f"--- [{r[iid]}] {r[ik][:90]}")
        if r[im] in WANT:
            print(f"    {r[im]:34s} {r[iv]} {r[iu]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr = rr[0]
    cols = [i for i, x in enumerate(hdr) if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued")]
    for r in rr[2:]:
        vals = []
        for i in cols:
            try:
                vals.append((float(r[i].replace(",", "")), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1
        top = sorted(vals, reverse=True)[:6]
        print(f"[{r[hdr.index('ID')]}] stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in top))


if __name__ == "__main__":
    main(sys.argv[1])
