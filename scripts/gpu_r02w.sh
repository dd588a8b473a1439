#!/bin/bash
# round 2: side columns (x walls' inner halo from dense side arrays) -- correctness, then timing
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/w_smoke.txt 2>&1; echo smoke=$? >> gpurun_out/w_smoke.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "side_columns or SC or XINTER or FASTDIV" > gpurun_out/t_w.log 2>&1
echo "rc=$?" >> gpurun_out/t_w.log
timeout 300 python scripts/ew_check.py C2 6 WAVE25_SC=0 > gpurun_out/ew_w.txt 2>&1
timeout 600 python scripts/ew_check.py C3 3 WAVE25_SC=0 >> gpurun_out/ew_w.txt 2>&1
for rep in 1 2; do
for cfg in "" "WAVE25_SC=0"; do
  echo "== $cfg" >> gpurun_out/qt_w.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_w.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_w.txt 2>&1
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_w.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_w.txt 2>&1
done
done
echo done
