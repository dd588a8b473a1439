#!/bin/bash
# round 2: C2 wall tiles (shorter x-wall tiles / two CTAs per SM) -- C2 has 4x fewer wall tile columns than C3
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hh_build.log 2>&1
for rep in 1 2; do
for cfg in "" "WAVE25_WALLX_TILE=x24c16x64x1r" "WAVE25_WALLX_TILE=x24c16x64x1r2" "WAVE25_WALLY_TILE=y128x8x1r2" "WAVE25_WALLX_TILE=x24c16x32x1"; do
  echo "== $cfg" >> gpurun_out/qt_hh.txt
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_hh.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_hh.txt 2>&1
done
done
echo done
