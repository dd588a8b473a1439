#!/bin/bash
# round 2: wall phases adjacent in time (walls last / first in the two steps of a graph), wall stores evict-normal
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y_build.log 2>&1
for rep in 1 2; do
for cfg in "" "WAVE25_WALLS_ALT=1" "WAVE25_WALLS_ALT=1 WAVE25_WALL_STKEEP=1" "WAVE25_WALL_STKEEP=1" "WAVE25_WALLS_LAST=1"; do
  echo "== $cfg" >> gpurun_out/qt_y.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_y.txt 2>&1
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_y.txt 2>&1
done
done
echo done
