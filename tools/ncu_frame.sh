#!/bin/bash
# ncu --set full capture of every kernel of one single-context frame (the 4th render
# of stage_timing's loop): bash tools/ncu_frame.sh [config] [tag]
# -> gpurun_out/frame_<tag>.ncu-rep and a per-kernel summary on stdout.
cfg=${1:-mip360}; tag=${2:-$cfg}
# kernels per frame: preprocess (3) + bin (~15) + blend (1); skip 3 warm-up frames
ncu --set full --import-source on --clock-control none -s 57 -c 19 -f -o gpurun_out/frame_$tag \
    python tools/stage_timing.py --config $cfg --iters 2 > gpurun_out/ncu_frame_$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/frame_$tag.ncu-rep
