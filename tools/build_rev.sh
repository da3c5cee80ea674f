#!/bin/bash
# Build libunimgs.so from a git revision (A/B baselines): tools/build_rev.sh <rev> <out.so> ["extra nvcc flags"]
# (rev WORKTREE: the working tree)
set -e
rev=$1; out=$(realpath -m "$2"); extra=${3:-}
d=$(mktemp -d)
if [ "$rev" = WORKTREE ]; then cp -r paper_2601_19233_b200 include "$d"/; else git archive "$rev" paper_2601_19233_b200/csrc include | tar -x -C "$d"; fi
cd "$d/paper_2601_19233_b200"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC,-fvisibility=hidden -shared --expt-relaxed-constexpr $extra -I"$d/include" -o "$out" \
  csrc/api.cu csrc/preprocess.cu csrc/binning.cu csrc/blend.cu csrc/deform.cu csrc/bind.cu
rm -rf "$d"
echo "$out"
