#!/bin/bash
# Per-kernel bin timings of one context (UNIMGS_BIN_EVENTS=1: CUDA events between launches), mip360 and nerf.
for cfg in mip360 nerf; do
UNIMGS_BIN_EVENTS=1 python tools/stage_timing.py --config $cfg --iters 20 2> /tmp/ev_$cfg.txt | tail -1 | cut -c1-160
python - $cfg <<'PY'
import sys, collections
cfg = sys.argv[1]
rows = [l.split() for l in open(f'/tmp/ev_{cfg}.txt') if l.startswith('bin_event')]
# per call sequence: find the number of marks per call (starts at 'scan+compact')
starts = [i for i, r in enumerate(rows) if r[1] == 'scan+compact']
per = starts[1] - starts[0]
calls = [rows[s:s + per] for s in starts[5:]]  # skip warm-up calls
agg = collections.OrderedDict()
for c in calls:
    for j, r in enumerate(c):
        agg.setdefault((j, r[1]), []).append(float(r[2]))
tot = 0
for (j, n), v in agg.items():
    m = sorted(v)[len(v) // 2]
    tot += m
    print(f"{cfg:7s} {j:2d} {n:16s} {m * 1000:8.1f} us")
print(f"{cfg:7s} total {tot * 1000:.1f} us over {len(calls)} calls")
PY
done
