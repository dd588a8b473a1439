#!/bin/bash
# time wall-kernel variants (development aid)
SC=${1:-C3}
for iv in ${INNER:-128x8x1}; do
for xv in ${WX:-x32x32x1 x32x64x2 x32x16x1}; do
  for yv in ${WY:-y128x16x1 y64x16x1}; do
    WAVE25_INNER_TILE=$iv WAVE25_WALLX_TILE=$xv WAVE25_WALLY_TILE=$yv timeout 300 python scripts/quick_time.py $SC stream 40 2>&1 | sed "s/^/$iv $xv $yv /" | tail -1
  done
done
done
