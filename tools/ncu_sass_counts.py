"""Executed-instruction profile of one kernel (SASS view of an ncu report):
total warp-instructions, average active lanes, and the most executed lines.

python tools/ncu_sass_counts.py report.ncu-rep <kernel regex> [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                                  text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
    h = rows[0]
    ie, te = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    src, ad = h.index("Source"), h.index("Address")
    data = []
    for r in rows[1:]:
        try:
            data.append((int(r[ie]), int(r[te]), r[ad], r[src].strip()))
        except (ValueError, IndexError):
            pass
    tw = sum(d[0] for d in data)
    tt = sum(d[1] for d in data)
    print(f"warp-instructions {tw:,}  thread-instructions {tt:,}  avg active lanes {tt / max(tw, 1):.1f}")
    for w, t, a, s in sorted(data, reverse=True)[:top]:
        print(f"{w:12,d} {t / max(w, 1):5.1f}  {a[-5:]}  {s[:110]}")


if __name__ == "__main__":
    main()
