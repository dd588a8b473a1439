#!/bin/bash
# round 2: table division (Markstein) + straight-line PML rows: timing A/B, bitwise variants, C3 x 1000 horizon
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "" "WAVE25_FASTDIV=0"; do
  echo "== $cfg" >> gpurun_out/qt_e.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_e.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_e.txt 2>&1
  env $cfg timeout 300 python scripts/quick_time.py C2 stream 200 >> gpurun_out/qt_e.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_e.txt 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or division or c2_full or edge or random" -p no:cacheprovider > gpurun_out/t_e.log 2>&1
echo "rc=$?" >> gpurun_out/t_e.log
WAVE25_SLOW=1 timeout 2400 python -m pytest tests/test_gpu_horizon.py -m gpu -x -q -s -k c3 -p no:cacheprovider > gpurun_out/t_c3h.log 2>&1
echo "rc=$?" >> gpurun_out/t_c3h.log
echo done
