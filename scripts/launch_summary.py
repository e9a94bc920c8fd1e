"""Per-kernel totals of an ncu launch list (``--metrics gpu__time_duration.sum --csv --log-file``).

    python scripts/launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import re
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[h + 1:]:
        v = float(r[iv].replace(",", ""))
        v = v / 1e6 if r[iu] == "ns" else (v / 1e3 if r[iu] in ("us", "usecond") else v)
        name = re.sub(r"\(.*$", "", r[ik].replace("(anonymous namespace)::", ""))
        name = re.sub(r"^void ", "", name)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{sum(cnt.values())} launches, {s:.3f} ms device time (ncu: cold cache, serialised)")
    print(f"{'kernel':45s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:45]:45s} {cnt[k]:8d} {v:10.3f} {100 * v / s:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
