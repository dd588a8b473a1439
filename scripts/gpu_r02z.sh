#!/bin/bash
# round 2: y walls with the interior's 248x8 tile shape
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "y248x8x1ry" > gpurun_out/t_z.log 2>&1; echo "rc=$?" >> gpurun_out/t_z.log
for rep in 1 2; do
for cfg in "" "WAVE25_WALLY_TILE=y248x8x1ry"; do
  echo "== $cfg" >> gpurun_out/qt_z.txt
  env $cfg timeout 120 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_z.txt 2>&1
  env $cfg timeout 120 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_z.txt 2>&1
  env $cfg timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_z.txt 2>&1
done
done
echo done
