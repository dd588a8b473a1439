#!/bin/bash
# round 2: C2 interior z-chunk length (default choose_cz: 86 planes, 720 units = 4.9 waves)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ff_build.log 2>&1
for cfg in "" "WAVE25_CZ=47" "WAVE25_CZ=64" "WAVE25_CZ=103" "WAVE25_CZ=128" "WAVE25_CZ=171" "WAVE25_CZ=256" "WAVE25_WALL_CZ=20" "WAVE25_WALL_CZ=40" ""; do
  echo "== $cfg" >> gpurun_out/qt_ff.txt
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_ff.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_ff.txt 2>&1
done
echo done
