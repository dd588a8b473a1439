#!/bin/bash
# round 2: interior z-chunk length and the 256-wide (line-aligned) tile re-measured at HEAD
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aa_build.log 2>&1
for cfg in "" "WAVE25_CZ=128" "WAVE25_CZ=171" "WAVE25_CZ=256" "WAVE25_CZ=342" "WAVE25_CZ=512" "WAVE25_INNER_TILE=256x8x1r" ""; do
  echo "== $cfg" >> gpurun_out/qt_aa.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_aa.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_aa.txt 2>&1
done
echo done
