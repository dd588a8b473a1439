#!/bin/bash
# round 2: 4-stage p ring for the x walls and the fp64 interior
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
  timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_j.txt 2>&1
  timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_j.txt 2>&1
  timeout 300 python scripts/quick_time.py C2 stream 200 >> gpurun_out/qt_j.txt 2>&1
done
timeout 300 python scripts/quick_time.py C3 stream 50 fp64 >> gpurun_out/qt_j.txt 2>&1
timeout 300 python scripts/prof_kinds.py C3 stream 6 fp64 >> gpurun_out/qt_j.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or edge or random or c1 or ragged" -p no:cacheprovider > gpurun_out/t_j.log 2>&1
echo "rc=$?" >> gpurun_out/t_j.log
echo done
