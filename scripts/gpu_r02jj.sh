#!/bin/bash
# round 2: fp64 x walls 16x32 with a producer warpgroup (no spills) vs 16x64 (spills)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/jj_build.log 2>&1
CHECK_PREC=fp64 timeout 300 python scripts/ew_check.py C2 6 WAVE25_DWALLX_TILE=dx24c16x32x1r > gpurun_out/jj_check.txt 2>&1
for rep in 1 2; do
for cfg in "" "WAVE25_DWALLX_TILE=dx24c16x32x1r"; do
  echo "== $cfg" >> gpurun_out/qt_jj.txt
  env $cfg timeout 200 python scripts/quick_time.py C3 stream 50 fp64 >> gpurun_out/qt_jj.txt 2>&1
  env $cfg timeout 200 python scripts/prof_kinds.py C3 stream 10 fp64 >> gpurun_out/qt_jj.txt 2>&1
done
done
echo done
