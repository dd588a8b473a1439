#!/bin/bash
# round 2: L2 promotion of the x-wall u boxes only (0 none, 1 64B, 3 256B; default 2 = 128B)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/kk_build.log 2>&1
for rep in 1 2; do
for cfg in "" "WAVE25_XWALL_UPROMO=3" "WAVE25_XWALL_UPROMO=1" "WAVE25_XWALL_UPROMO=0"; do
  echo "== $cfg" >> gpurun_out/qt_kk.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_kk.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_kk.txt 2>&1
done
done
echo done
