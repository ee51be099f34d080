#!/usr/bin/env bash
# Build library variants that differ in compile-time knobs (nvcc -D...) for
# A/B runs on the GPU box:
#
#   tools/ab_build.sh "c4:-DWD_LDA_MIN_BLOCKS_COARSE=4" "c6:-DWD_LDA_MIN_BLOCKS_COARSE=6"
#   # then, on the box, per variant:
#   WARPDRAW_B200_LIB=paper_1505_03851_b200/_lib/var/libwd_c4.so python tools/configs.py --only cfg5_shard
#
# Knobs (wd_draw.cuh): WD_LDA_MIN_BLOCKS, WD_LDA_MIN_BLOCKS_COARSE,
# WD_LDA_MIN_BLOCKS_F64, WD_MIN_BLOCKS_OTHER.  Runtime knobs (wd_launch.cuh):
# WD_PIPE_ROWS / WD_PIPE_LDA (block-loop variant), WD_L2_X / WD_L2_T (L2
# eviction policy of the phi / theta loads).  Delete _lib/var before the
# final snapshot: variants travel with gpurun.
set -euo pipefail
cd "$(dirname "$0")/.."
mkdir -p paper_1505_03851_b200/_lib/var
for spec in "$@"; do
  name="${spec%%:*}"
  flags="${spec#*:}"
  WD_LIB_OUT="paper_1505_03851_b200/_lib/var/libwd_${name}.so" WD_EXTRA_FLAGS="$flags" \
    python -m paper_1505_03851_b200.build --force > "/tmp/ab_build_${name}.log" 2>&1 &
done
wait
ls -la paper_1505_03851_b200/_lib/var/*.so
