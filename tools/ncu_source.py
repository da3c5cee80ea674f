"""Per-source-line (or SASS) stall samples of one kernel from an ncu report.

python tools/ncu_source.py report.ncu-rep <kernel regex> [--sass] [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    sass = "--sass" in sys.argv
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"]
    out = subprocess.check_output(cmd, text=True, stderr=subprocess.DEVNULL)
    lines = out.splitlines()
    # several launches may match: keep the section of the --nth one (default 0)
    nth = int(sys.argv[sys.argv.index("--nth") + 1]) if "--nth" in sys.argv else 0
    starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
    lines = lines[starts[nth]:starts[nth + 1]]
    print(lines[0][:160])
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    loc = h.index("Address") if "Address" in h else (h.index("# Line") if "# Line" in h else 0)
    data = []
    for r in rows[1:]:
        if len(r) <= si:
            continue
        try:
            v = float(r[si])
        except ValueError:
            continue
        data.append((v, r[loc], r[src].strip()))
    tot = sum(d[0] for d in data) or 1
    for v, a, s in sorted(data, reverse=True)[:top]:
        print(f"{100 * v / tot:5.1f}%  {a:>10s}  {s[:150]}")


if __name__ == "__main__":
    main()
