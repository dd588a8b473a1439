#!/bin/bash
# round 2: packed fp32 Laplacian in the y-wall kernel (A/B build libwave25_packy.so)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1
for rep in 1 2; do
for cfg in "" "WAVE25_LIB=libwave25_packy.so"; do
  echo "== $cfg" >> gpurun_out/qt_s.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_s.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_s.txt 2>&1
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_s.txt 2>&1
done
done
WAVE25_LIB=libwave25_packy.so timeout 300 python scripts/ew_check.py C2 6 WAVE25_LIB=libwave25_packy.so >> gpurun_out/qt_s.txt 2>&1
echo done
