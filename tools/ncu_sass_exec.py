"""SASS listing of one kernel from an ncu report with per-instruction warp-level
executions, average active threads and stall samples (the hot loop at a glance).

python tools/ncu_sass_exec.py report.ncu-rep [kernel regex] [--min N] [--skip K]
(--skip K: the K-th launch matching the regex, 0-based)
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "."
    mn = float(sys.argv[sys.argv.index("--min") + 1]) if "--min" in sys.argv else 0
    skip = sys.argv[sys.argv.index("--skip") + 1] if "--skip" in sys.argv else "0"
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                                   "-k", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                                  text=True, stderr=subprocess.DEVNULL)
    lines = out.splitlines()
    starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
    print(lines[starts[0]][:140])
    rows = list(csv.reader(io.StringIO("\n".join(lines[starts[0] + 1:starts[1]]))))
    h = rows[0]
    ie, th, ss, src = (h.index("Instructions Executed"), h.index("Avg. Threads Executed"),
                       h.index("Warp Stall Sampling (All Samples)"), h.index("Source"))
    tot = sum(float(r[ie] or 0) for r in rows[1:] if len(r) > ie)
    samp = sum(float(r[ss] or 0) for r in rows[1:] if len(r) > ss)
    print(f"total warp-instructions {tot / 1e6:.1f} M, stall samples {samp:.0f}")
    for i, r in enumerate(rows[1:]):
        if len(r) <= ie:
            continue
        n = float(r[ie] or 0)
        if n < mn:
            continue
        print(f"{i:5d} {n / 1e6:8.3f}M {float(r[th] or 0):5.1f}t {float(r[ss] or 0):6.0f}s  {r[src].strip()}")


if __name__ == "__main__":
    main()
