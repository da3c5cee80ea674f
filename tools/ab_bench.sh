#!/bin/bash
# A/B the bench's device-timed frames/s between the in-tree library and experiment builds.
for rep in 1 2; do
  for L in "" "$@"; do
    if [ -z "$L" ]; then env -u UNIMGS_LIB python bench.py --no-e2e --no-cpu-baseline $BENCH_ARGS
    else UNIMGS_LIB=$L python bench.py --no-e2e --no-cpu-baseline $BENCH_ARGS; fi 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', 'fps %.1f frame_ms %.4f blend_in_region %.4f' % (d['value'], d['frame_ms'], d['roofline']['avg_launch_ms']))"
  done
done
