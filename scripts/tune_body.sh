#!/bin/bash
# time body/wall tile variants on one scenario (development aid)
SC=${1:-C3}
for v in ${BODY:-128x8x1 128x16x1 64x16x1 128x8x2 256x8x1}; do
  for wv in ${WALL:-w128x16x1}; do
    WAVE25_WALL_TILE=$wv WAVE25_BODY_TILE=$v timeout 300 python scripts/quick_time.py $SC stream 40 2>&1 | sed "s/^/$v $wv /" | tail -1
  done
done
