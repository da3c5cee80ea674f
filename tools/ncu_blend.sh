#!/bin/bash
# ncu --set full capture of one k_blend launch (mip360 view 0, the 4th render) for each
# library given (in-tree when none): bash tools/ncu_blend.sh [config] [lib ...]
# Reports land in gpurun_out/blend_<tag>.ncu-rep and a summary on stdout.
cfg=${1:-mip360}; shift
libs=("$@"); [ ${#libs[@]} -eq 0 ] && libs=("")
for L in "${libs[@]}"; do
  tag=$(basename "${L:-intree}" .so)_$cfg
  if [ -z "$L" ]; then envs="env -u UNIMGS_LIB"; else envs="env UNIMGS_LIB=$L"; fi
  $envs ncu --set full --import-source on --clock-control none -k regex:k_blend -s 3 -c 1 -f \
      -o gpurun_out/blend_$tag python tools/stage_timing.py --config $cfg --iters 2 > gpurun_out/ncu_$tag.log 2>&1
  echo "== $tag"; python tools/ncu_summary.py gpurun_out/blend_$tag.ncu-rep 2>&1 | head -40
done
