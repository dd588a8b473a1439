#!/bin/bash
# round 2: zero-select table division timing A/B; interior chunk/prefetch sweep; wall ncu
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "" "WAVE25_FASTDIV=0"; do
  echo "== $cfg" >> gpurun_out/qt_g.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_g.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_g.txt 2>&1
  env $cfg timeout 300 python scripts/quick_time.py C2 stream 200 >> gpurun_out/qt_g.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_g.txt 2>&1
done
for cz in 103 128 171 205; do
  echo "== CZ $cz" >> gpurun_out/qt_g.txt
  WAVE25_CZ=$cz timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_g.txt 2>&1
done
for pf in 0 2; do
  echo "== PF $pf" >> gpurun_out/qt_g.txt
  WAVE25_PF=$pf timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_g.txt 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_stream<(24|128)," -s 2 -c 2 -o gpurun_out/prof_g python scripts/prof_kinds.py C3 stream 1 > gpurun_out/ncu_g.log 2>&1
echo done
