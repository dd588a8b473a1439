#!/bin/bash
# round 2: seam x walls: correctness first, then timing and ncu
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_point or c1_random or edge or variants" -p no:cacheprovider > gpurun_out/t_k1.log 2>&1
echo "rc=$?" >> gpurun_out/t_k1.log
for cfg in "" "WAVE25_SEAM=0"; do
  echo "== $cfg" >> gpurun_out/qt_k.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_k.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_k.txt 2>&1
  env $cfg timeout 300 python scripts/quick_time.py C2 stream 200 >> gpurun_out/qt_k.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_k.txt 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_stream<\(int\)(32|128),' -s 2 -c 2 -o gpurun_out/prof_k python scripts/prof_kinds.py C3 stream 1 > gpurun_out/ncu_k.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_horizon.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_k2.log 2>&1
echo "rc=$?" >> gpurun_out/t_k2.log
echo done
