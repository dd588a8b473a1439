#!/bin/bash
# round 2: stored-eta wall tiles (producer-warpgroup shapes) vs the defaults
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dd_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_eta.py -m gpu -q -p no:cacheprovider -k "variants" > gpurun_out/t_dd.log 2>&1; echo "rc=$?" >> gpurun_out/t_dd.log
for rep in 1 2; do
for cfg in "" "WAVE25_EWALLY_TILE=ey128x16x1r" "WAVE25_EWALLY_TILE=ey128x8x1r" "WAVE25_EWALLX_TILE=ex24c16x64x1r"; do
  echo "== $cfg" >> gpurun_out/qt_dd.txt
  env $cfg PROF_ETA=1 timeout 200 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_dd.txt 2>&1
done
done
echo done
