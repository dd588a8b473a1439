#!/bin/bash
# round 2: per-geometry interior tile (C2 -> 240), full -m gpu suite
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v_smoke.txt 2>&1; echo smoke=$? >> gpurun_out/v_smoke.txt
timeout 120 python scripts/quick_time.py C3 stream 200 > gpurun_out/qt_v.txt 2>&1
timeout 120 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_v.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_v.log 2>&1
echo "rc=$?" >> gpurun_out/t_v.log
echo done
