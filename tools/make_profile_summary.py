"""Write the committed profile evidence of a round from gpurun_out/ artefacts.

python tools/make_profile_summary.py <tag> <launches.csv> <frame.ncu-rep> <bench.json> [<ref.json>]

Produces profiles/<tag>_summary.md, profiles/<tag>_launches.csv (copy),
profiles/<tag>_ncu_full.csv (raw metrics of the full capture) and
profiles/blend_traffic.json (DRAM bytes per k_blend launch, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import raw, fnum  # noqa: E402


def launch_shares(path):
    """Per kernel name: launches, mean duration, and launches per frame (frames =
    k_begin_frame launches; the warm-up, timed, isolated and counting passes of the
    bench command all render whole frames, so per-frame averages are comparable)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("unimgs::", "")
        per.setdefault(name, []).append(float(r[vi].replace(",", "")))
    frames = max(1, len(per.get("k_begin_frame", [])))
    return per, frames


def main():
    tag, lpath, rep, bpath = sys.argv[1:5]
    ref = sys.argv[5] if len(sys.argv) > 5 else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    shutil.copy(lpath, os.path.join(ROOT, "profiles", f"{tag}_launches.csv"))
    bench = json.load(open(bpath))
    per, frames = launch_shares(lpath)
    cmd = os.environ.get("PROFILE_CMD", "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline")
    frame_us = {k: sum(v) / frames for k, v in per.items()}
    tot = sum(frame_us.values())
    lines = [f"# {tag}: ncu evidence for the bench line", ""]
    lines += ["## Bench line (bench.py, 1 GPU)", "", "```json", json.dumps(bench, indent=1)[:6000], "```", ""]
    if ref and os.path.exists(ref):
        lines += ["## Reference arm (CPU oracle)", "", "```json", open(ref).read().strip(), "```", ""]
    lines += ["## Launch list: kernel shares of a frame (ncu gpu__time_duration, cold-cache, serialised)", "",
              f"Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv {cmd}`; "
              f"{frames} frames (k_begin_frame launches) over the warm-up, timed, isolated-blend and "
              "work-counting passes; `k_blend<1,...>` is the counting variant of the last pass.  The bench's "
              "4 concurrent contexts run the sort passes at 1 CTA/SM (`settings.sort_ctas_per_sm`, which leaves "
              "the rest of each SM to the other contexts' blends), so serialised under ncu they show their "
              "stand-alone latency; the full capture below is one frame of a single context (4 CTAs/SM).", "",
              "| kernel | launches | mean us | us per frame | share of frame |", "|---|---|---|---|---|"]
    for k, v in per.items():
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {frame_us[k] / 1e3:.1f} | "
                     f"{frame_us[k] / tot:.3f} |")
    lines.append("")
    rows = raw(rep)
    lines += ["## Full capture of one mip360 frame (`ncu --set full`)", "",
              "| kernel | us | DRAM MB r+w | DRAM % peak | warps active % | issue % active | regs |",
              "|---|---|---|---|---|---|---|"]
    blend = None
    for d in rows:
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        t = fnum(d["gpu__time_duration.sum"])
        mb = (fnum(d["dram__bytes_read.sum"]) + fnum(d["dram__bytes_write.sum"]))
        lines.append(f"| {name} | {t:.1f} | {mb:.1f} | {d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']} | "
                     f"{d['sm__warps_active.avg.pct_of_peak_sustained_active']} | "
                     f"{d['sm__inst_issued.avg.pct_of_peak_sustained_active']} | {d['launch__registers_per_thread']} |")
        if name.startswith("unimgs::k_blend") or name.startswith("k_blend"):
            issue_active = fnum(d["sm__inst_issued.avg.pct_of_peak_sustained_active"])
            cyc_act, cyc_el = fnum(d.get("smsp__cycles_active.avg", "nan")), fnum(d.get("sm__cycles_elapsed.avg", "nan"))
            blend = {"kernel": name, "dram_bytes_per_launch": mb * 1e6, "duration_us_ncu": t,
                     "issue_active_pct": issue_active,
                     "sm_active_frac": cyc_act / cyc_el if cyc_el == cyc_el and cyc_el > 0 else None,
                     "issue_elapsed_pct": issue_active * cyc_act / cyc_el if cyc_el == cyc_el and cyc_el > 0 else None,
                     "source": f"profiles/{tag}_ncu_full.csv"}
    lines.append("")
    lines.append("DRAM MB are ncu's `dram__bytes_read.sum + dram__bytes_write.sum` (units as reported: MB).")
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.csv"), "w").write(out)
    if blend:
        json.dump(blend, open(os.path.join(ROOT, "profiles", "blend_traffic.json"), "w"), indent=1)
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
