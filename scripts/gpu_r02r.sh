#!/bin/bash
# round 2: embedded wall warps -- where the time goes (wall per-plane time during the interior vs mop-up)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r_build.log 2>&1
for cfg in "WAVE25_EW_PF=0" "WAVE25_EW_PF=8" "WAVE25_EW_PF=16" "WAVE25_EW_PF=8 WAVE25_EW_CZ=200" "WAVE25_EW_PF=8 WAVE25_EW_REM=1000000"; do
  echo "== $cfg" >> gpurun_out/qt_r.txt
  env $cfg timeout 120 python scripts/ew_probe.py C3 20 >> gpurun_out/qt_r.txt 2>&1
done
echo done
