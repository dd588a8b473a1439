#!/bin/bash
# round 2: packed-fp32 A/B, stored-eta TMA staging, wall/interior ncu --set full
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_eta.py tests/test_gpu_fp64.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_eta.log 2>&1
echo "rc=$?" >> gpurun_out/t_eta.log
for lib in "" "WAVE25_LIB=libwave25_scalar.so"; do
  echo "== $lib" >> gpurun_out/qt_d.txt
  env $lib timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_d.txt 2>&1
  env $lib timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_d.txt 2>&1
  env $lib timeout 300 python scripts/quick_time.py C2 stream 200 >> gpurun_out/qt_d.txt 2>&1
  env $lib PROF_ETA=1 timeout 300 python scripts/prof_kinds.py C3 stream 6 >> gpurun_out/qt_d.txt 2>&1
done
for t in 128x16x1 248x8x2; do
  echo "== tile $t" >> gpurun_out/qt_d.txt
  WAVE25_INNER_TILE=$t timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_d.txt 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stream -s 3 -c 3 -o gpurun_out/prof_d python scripts/prof_kinds.py C3 stream 2 > gpurun_out/ncu_d.log 2>&1
echo done
