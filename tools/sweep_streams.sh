#!/bin/bash
# Bench frames/s versus the number of concurrent contexts/streams (4 is the default).
for n in 2 3 4 6 8; do
  python bench.py --no-e2e --no-cpu-baseline --streams $n 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('streams $n', 'fps %.1f' % d['value'])"
done
