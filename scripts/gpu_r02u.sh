#!/bin/bash
# round 2: C2 interior tile width (480 = 2 x 240)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u_build.log 2>&1
for rep in 1 2; do
for cfg in "" "WAVE25_INNER_TILE=240x8x1r" "WAVE25_INNER_TILE=256x8x1r"; do
  echo "== $cfg" >> gpurun_out/qt_u.txt
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_u.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_u.txt 2>&1
done
done
echo done
