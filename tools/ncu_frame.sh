#!/bin/bash
# ncu --set full capture of every kernel of one single-context frame (the 4th frame
# of stage_timing's loop): bash tools/ncu_frame.sh [config] [tag]
# -> gpurun_out/frame_<tag>.ncu-rep and a per-kernel summary on stdout.
cfg=${1:-mip360}; tag=${2:-$cfg}
# the frame's kernels (sort_mode 0): begin, B2, B1, scan + compact, hist, 4 depth
# passes, dup count + scan, range starts, expand, 2 x (count +) scan + downsweep,
# ranges, order, blend = 22 launches; skip 3 frames
K='regex:k_(begin_frame|setup_triangles|preprocess_gaussians|scan_counts|compact|hist_depth|onesweep|dup_count|range_starts|expand|rts_scan|downsweep|tile_count|ranges16|tile_order|blend)'
ncu --set full --import-source on --clock-control none -k "$K" -s 66 -c 22 -f -o gpurun_out/frame_$tag \
    python tools/stage_timing.py --config $cfg --iters 5 > gpurun_out/ncu_frame_$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/frame_$tag.ncu-rep
