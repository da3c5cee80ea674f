"""Summarise an ncu --set full report: per-kernel duration, DRAM bytes, occupancy,
issue utilisation and the top warp-stall reasons (markdown on stdout).

python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["smsp__cycles_active.avg", "sm__cycles_elapsed.avg", 
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "lts__t_sector_hit_rate.pct",
    "smsp__inst_executed.sum",
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "not_selected", "selected", "no_instruction", "dispatch_stall", "branch_resolving",
          "membar", "sleeping", "drain", "imc_miss", "tex_throttle", "misc"]


def raw(report):
    names = METRICS + [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]
    out = subprocess.check_output(["ncu", "-i", report, "--page", "raw", "--csv", "--metrics", ",".join(names)],
                                  text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        res.append(d)
    return res


def fnum(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    rep = sys.argv[1]
    rows = raw(rep)
    out = []
    print(f"| kernel | us | DRAM MB (r+w) | DRAM % | warps active % | issue % | regs | warp-inst (M) | top stalls (warps/issue) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for d in rows:
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        us = fnum(d["gpu__time_duration.sum"]) / (1e3 if fnum(d["gpu__time_duration.sum"]) > 1e4 else 1)
        mb = fnum(d["dram__bytes_read.sum"]) + fnum(d["dram__bytes_write.sum"])
        st = sorted(((fnum(d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", "nan")), s)
                     for s in STALLS), reverse=True)[:3]
        top = ", ".join(f"{s} {v:.2f}" for v, s in st if v == v)
        print(f"| {name} | {d['gpu__time_duration.sum']} | {mb:.1f} | {d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']} | "
              f"{d['sm__warps_active.avg.pct_of_peak_sustained_active']} | {d['sm__inst_issued.avg.pct_of_peak_sustained_active']} | "
              f"{d['launch__registers_per_thread']} | {fnum(d['smsp__inst_executed.sum']) / 1e6:.1f} | {top} |")
        out.append({"kernel": name, **{k: d.get(k) for k in METRICS},
                    "stalls": {s: v for v, s in st}})
    if "--json" in sys.argv:
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
