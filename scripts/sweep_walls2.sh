#!/bin/bash
for xv in x24c16x32x1 x24c16x32x1m3 x24c16x32x1m4; do for yv in y128x8x1 y128x8x1m2 y64x8x1m3; do
  WAVE25_WALLX_TILE=$xv WAVE25_WALLY_TILE=$yv timeout 300 python scripts/quick_time.py C3 stream 60 2>&1 | sed "s/^/$xv $yv /" | tail -1
done; done
