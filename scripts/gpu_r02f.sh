#!/bin/bash
# round 2: swizzled x walls + unpacked walls + eta staging fix: correctness, timing, ncu of the walls
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_eta.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_f_eta.log 2>&1
echo "rc=$?" >> gpurun_out/t_f_eta.log
for cfg in "" "WAVE25_FASTDIV=0"; do
  echo "== $cfg" >> gpurun_out/qt_f.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_f.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_f.txt 2>&1
  env $cfg timeout 300 python scripts/quick_time.py C2 stream 200 >> gpurun_out/qt_f.txt 2>&1
done
for t in y248x8x1r y128x16x1rg; do echo "== ytile $t" >> gpurun_out/qt_f.txt; WAVE25_WALLY_TILE=$t timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_f.txt 2>&1; done
echo "== xtile g" >> gpurun_out/qt_f.txt; WAVE25_WALLX_TILE=x24c16x128x1rg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_f.txt 2>&1
echo "== eta" >> gpurun_out/qt_f.txt
PROF_ETA=1 timeout 300 python scripts/prof_kinds.py C3 stream 6 >> gpurun_out/qt_f.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream<(24|128)," -s 2 -c 2 -o gpurun_out/prof_f python scripts/prof_kinds.py C3 stream 1 > gpurun_out/ncu_f.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tb2.py tests/test_gpu_pair.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_f.log 2>&1
echo "rc=$?" >> gpurun_out/t_f.log
echo done
