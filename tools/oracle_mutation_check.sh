#!/usr/bin/env bash
# Mutation check of the oracle's pins: each mutation is applied to a scratch copy of
# the repo and the CPU pin suites must FAIL on it.  Usage: tools/oracle_mutation_check.sh
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PINS="tests/test_oracle_pins.py tests/test_oracle_shading_pins.py tests/test_oracle_modes.py tests/test_oracle_tri_depth.py tests/test_oracle_degenerate.py tests/test_oracle_resort.py tests/test_oracle_fragment_counts.py"
declare -a MUT=(
  # name|sed expression on oracle/unimgs_oracle.c
  'bilinear_t10_t01|s/double t00 = texel(c, i0, j0, ch), t10 = texel(c, i0 + 1, j0, ch);/double t00 = texel(c, i0, j0, ch), t10 = texel(c, i0, j0 + 1, ch);/; s/double t01 = texel(c, i0, j0 + 1, ch), t11/double t01 = texel(c, i0 + 1, j0, ch), t11/'
  'sh_dir_reversed|s/d\[a\] = (double)c->means\[3 \* i + a\] - cp\[a\];/d[a] = cp[a] - (double)c->means[3 * i + a];/'
  'fov_lx_from_height|s/float lx = 1.3f \* (0.5f \* (float)cam->width \/ cam->fx);/float lx = 1.3f * (0.5f * (float)cam->height \/ cam->fx);/'
  'fov_no_clamp|s/float tx = fminf(fmaxf(xz, -lx), lx) \* pv\[2\];/float tx = xz * pv[2];/'
  'texel_no_centre_offset|s/double tx = uu \* c->tw - 0.5, ty = vv \* c->th - 0.5;/double tx = uu * c->tw, ty = vv * c->th;/'
  'resort_pops_largest|s/        if (frag_pless(\&win->w\[i\], \&win->w\[m\])) m = i;/        if (frag_pless(\&win->w[m], \&win->w[i])) m = i;/'
  'resort_ties_by_larger_id|s/return da != db ? da < db : a->id < b->id;/return da != db ? da < db : a->id > b->id;/'
  'pixel_depth_at_corner|s/return or_tri_point_depth(c, f, 256 \* (int64_t)x + 128, 256 \* (int64_t)y + 128);/return or_tri_point_depth(c, f, 256 * (int64_t)x, 256 * (int64_t)y);/'
  'counts_kind_swapped|s/cnt\[apply->kind == 0 ? 0 : 1\]++;/cnt[apply->kind == 0 ? 1 : 0]++;/'
)
rc=0
for m in "${MUT[@]}"; do
  name=${m%%|*}; expr=${m#*|}
  d=/tmp/oracle_mut_$name
  rm -rf "$d"; mkdir -p "$d"
  (cd "$ROOT" && tar --exclude=.git --exclude=gpurun_out --exclude='*.so' -cf - oracle tests paper_2601_19233_b200/scenes.py paper_2601_19233_b200/__init__.py pytest.ini) | (cd "$d" && tar xf -)
  cp "$d/oracle/unimgs_oracle.c" "$d/orig.c"
  sed -i "$expr" "$d/oracle/unimgs_oracle.c"
  if cmp -s "$d/orig.c" "$d/oracle/unimgs_oracle.c"; then echo "$name: MUTATION NOT APPLIED"; rc=1; continue; fi
  if (cd "$d" && timeout 900 python -m pytest $PINS -x -q -m "not gpu" -p no:cacheprovider > log.txt 2>&1); then
    echo "$name: SURVIVED (no pin fails)"; rc=1
  else
    echo "$name: killed by $(grep -m1 -o 'FAILED [^ ]*' "$d/log.txt")"
  fi
done
exit $rc
