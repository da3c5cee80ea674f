#!/bin/bash
# A/B the per-stage device times between the in-tree library and experiment builds:
#   bash tools/ab_blend.sh exp/lib_a.so exp/lib_b.so   (in-tree first, twice each)
for rep in 1 2; do
  for L in "" "$@"; do
    for c in stress mip360 nerf; do
      if [ -z "$L" ]; then env -u UNIMGS_LIB python tools/stage_timing.py --config $c --iters 50
      else UNIMGS_LIB=$L python tools/stage_timing.py --config $c --iters 50; fi |
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['config'], 'pre %.4f bin %.4f blend %.4f' % (d['preprocess_ms'], d['bin_ms'], d['render_ms']))"
    done
  done
done
