"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python scripts/ncu_summary.py gpurun_out/launches.csv [--last K]

Groups launches by kernel (template args kept), prints count, total and
share of device time.  `--last K` restricts to the last K engine launches of
the timed step (the bench prints gpu_launches per step).
"""

import argparse
import csv
import io
import re


def load(path):
    text = open(path).read().splitlines()
    start = next(i for i, line in enumerate(text) if line.startswith('"ID"'))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(text[start:]))) if r.get("ID", "").isdigit()]
    return rows


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("uh::<unnamed>::", "").replace("void ", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--last", type=int, default=0)
    ap.add_argument("--skip-prefix", default="k_imad_peak,k_mac_peak,k_macc_peak,k_mulmod_peak,k_shoup_peak")
    args = ap.parse_args()
    rows = load(args.csv)
    skip = tuple(args.skip_prefix.split(","))
    rows = [r for r in rows if not short(r["Kernel Name"]).startswith(skip)
            and not short(r["Kernel Name"]).split("<")[0].endswith("_peak")
            and not short(r["Kernel Name"]).startswith(("at::", "regular_fft", "vector_fft"))]
    if args.last:
        rows = rows[-args.last:]
    agg = {}
    for r in rows:
        k = short(r["Kernel Name"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"]) / 1e3
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total / 1e3:.3f} ms device time (ncu: cold cache, serialised)")
    print(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:34s} {n:8d} {us / 1e3:10.3f} {100 * us / total:6.1f}%")


if __name__ == "__main__":
    main()
