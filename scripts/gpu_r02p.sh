#!/bin/bash
# round 2: premise of embedded wall warps: interior with a 3-stage u_prev/vdt2 ring, consumers at 104 registers
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1
for cfg in "" "WAVE25_LIB=libwave25_sp3.so" "WAVE25_INNER_TILE=248x8x1r104" "WAVE25_LIB=libwave25_sp3.so WAVE25_INNER_TILE=248x8x1r104"; do
  echo "== $cfg" >> gpurun_out/qt_p.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_p.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_p.txt 2>&1
done
echo done
