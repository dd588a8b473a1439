#!/bin/bash
# round 2: two CTAs per SM (producer warpgroup + 8 consumer warps at 104 registers each) -- interior and walls
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
for cfg in "" "WAVE25_INNER_TILE=128x8x1r2" "WAVE25_INNER_TILE=c124x8x1r2" "WAVE25_WALLX_TILE=x24c16x64x1r2" "WAVE25_WALLY_TILE=y128x8x1r2" "WAVE25_WALLX_TILE=x24c16x64x1r2 WAVE25_WALLY_TILE=y128x8x1r2"; do
  echo "== $cfg" >> gpurun_out/qt_t.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_t.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_t.txt 2>&1
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_t.txt 2>&1
done
echo done
