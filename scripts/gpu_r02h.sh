#!/bin/bash
# round 2: wall kernels under ncu (stall reasons, TMA / L2 / smem), x-wall tile variants
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for t in x24c16x128x1r x24c16x64x1r x24c16x32x1 x24c16x64x1; do
  echo "== xtile $t" >> gpurun_out/qt_h.txt
  WAVE25_WALLX_TILE=$t timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_h.txt 2>&1
  WAVE25_WALLX_TILE=$t timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_h.txt 2>&1
done
for t in y128x16x1r y64x16x1m2 y128x8x1m3; do
  echo "== ytile $t" >> gpurun_out/qt_h.txt
  WAVE25_WALLY_TILE=$t timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_h.txt 2>&1
  WAVE25_WALLY_TILE=$t timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_h.txt 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_stream<\(int\)(24|128),' -s 2 -c 2 -o gpurun_out/prof_h python scripts/prof_kinds.py C3 stream 1 > gpurun_out/ncu_h.log 2>&1
echo done
