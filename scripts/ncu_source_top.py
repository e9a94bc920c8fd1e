"""Top stalled SASS instructions of one kernel in an ncu report (needs --import-source / -lineinfo).

    python scripts/ncu_source_top.py REPORT KERNEL_REGEX [N] [LAUNCH]
"""
import csv
import io
import subprocess
import sys


def main(path, kern, n=20, which=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kern}", "--launch-skip", str(which), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, iw = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    sections, data = [], []
    for r in rows[2:]:
        if len(r) != len(hdr) or not r[iw].isdigit():
            if data:
                sections.append(data)
                data = []
            continue
        data.append(r)
    if data:
        sections.append(data)
    data = sections[0]
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[iw]) for r in data) or 1
    print(f"{len(data)} SASS lines, {tot} samples")
    order = sorted(range(len(data)), key=lambda k: -int(data[k][iw]))[:n]
    for k in order:
        r = data[k]
        st = sorted([(int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in sc], reverse=True)[:2]
        print(f"{k:5d} {100 * int(r[iw]) / tot:5.1f}% {r[ia][:64]:64s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 20,
         int(sys.argv[4]) if len(sys.argv) > 4 else 0)
