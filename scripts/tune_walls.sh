#!/bin/bash
# time kernel-variant combinations (development aid)
SC=${1:-C3}
for iv in ${INNER:-128x8x1}; do
for xv in ${WX:-x32c16x32x1}; do
  for yv in ${WY:-y128x8x1}; do
   for pr in ${PRIO:-1}; do
    WAVE25_WALL_PRIO=$pr WAVE25_INNER_TILE=$iv WAVE25_WALLX_TILE=$xv WAVE25_WALLY_TILE=$yv timeout 300 python scripts/quick_time.py $SC stream 40 2>&1 | sed "s/^/$iv $xv $yv prio=$pr /" | tail -1
   done
  done
done
done
