#!/bin/bash
# time interior-tile variants x L2-prefetch distances on one scenario (development aid)
SC=${1:-C3}
for v in ${VARIANTS:-64x32x2 64x16x2 64x16x1 64x32x1 128x16x1 128x16x2 128x8x1}; do
  for pf in ${PFS:-0 2 4}; do
    WAVE25_PF=$pf WAVE25_INNER_TILE=$v timeout 300 python scripts/quick_time.py $SC stream 40 2>&1 | sed "s/^/$v pf=$pf /" | tail -1
  done
done
