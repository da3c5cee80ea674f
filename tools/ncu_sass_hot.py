"""SASS of one kernel in address order with executed-instruction counts (hot lines only).

python tools/ncu_sass_hot.py report.ncu-rep <kernel regex> [--min FRACTION]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    mn = float(sys.argv[sys.argv.index("--min") + 1]) if "--min" in sys.argv else 0.002
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                                   "-k", f"regex:{kern}"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1] if rows[0][0] == "Kernel Name" else rows[0]
    body = rows[2:] if rows[0][0] == "Kernel Name" else rows[1:]
    ie, th, src = h.index("Instructions Executed"), h.index("Avg. Threads Executed"), h.index("Source")
    data = [(int(r[ie] or 0), r[th], r[src].strip()) for r in body if len(r) > ie]
    tot = sum(d[0] for d in data)
    print(f"total warp instructions {tot:,}")
    for n, t, s in data:
        if n >= mn * tot / 100:
            print(f"{100 * n / tot:6.2f}% {n:>11,} thr {t:>5}  {s}")


if __name__ == "__main__":
    main()
