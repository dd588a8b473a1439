#!/bin/bash
# combined knob sweep on C3 (development aid)
for yv in y128x8x1 y128x16x1; do for pf in 1 2 3; do for cz in 0 128; do
  E="WAVE25_WALLY_TILE=$yv WAVE25_PF=$pf"; [ $cz -gt 0 ] && E="$E WAVE25_CZ=$cz"
  env $E timeout 300 python scripts/quick_time.py C3 stream 60 2>&1 | sed "s/^/$yv pf=$pf cz=$cz /" | tail -1
done; done; done
