"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.

python tools/kernel_times.py launches.csv [--skip-first N]
"""
import collections
import csv
import sys


def main(path, skip=0):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1 + skip:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':44s} {'n':>4s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
    for k, v in agg.items():
        print(f"{k:44s} {len(v):4d} {sum(v)/len(v)/1e3:9.1f} {sum(v)/1e3:10.1f} {sum(v)/tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
