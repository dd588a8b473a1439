#!/bin/bash
# round 2: embedded wall warps (MODE_INNER_EW) -- correctness first, then timing
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "variants and EW" > gpurun_out/t_q.log 2>&1
echo "rc=$?" >> gpurun_out/t_q.log
timeout 300 python scripts/ew_check.py C2 6 WAVE25_EW=1 > gpurun_out/ew_q.txt 2>&1
timeout 600 python scripts/ew_check.py C3 3 WAVE25_EW=1 >> gpurun_out/ew_q.txt 2>&1
for cfg in "" "WAVE25_EW=1" "WAVE25_EW=1 WAVE25_EW_CZ=32" "WAVE25_EW=1 WAVE25_EW_CZ=128" "WAVE25_EW=1 WAVE25_EW_REM=0"; do
  echo "== $cfg" >> gpurun_out/qt_q.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_q.txt 2>&1
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_q.txt 2>&1
done
echo done
