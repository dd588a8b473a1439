#!/bin/bash
# round 2: stored-eta parity with the new default wall shapes
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ee_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_eta.py tests/test_gpu_fp64.py -m gpu -q -p no:cacheprovider > gpurun_out/t_ee.log 2>&1; echo "rc=$?" >> gpurun_out/t_ee.log
PROF_ETA=1 timeout 200 python scripts/prof_kinds.py C3 stream 10 > gpurun_out/qt_ee.txt 2>&1
echo done
