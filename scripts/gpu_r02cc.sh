#!/bin/bash
# round 2 end: smoke + full -m gpu suite at HEAD
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/cc_smoke.txt 2>&1; echo smoke=$? >> gpurun_out/cc_smoke.txt
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_cc.log 2>&1
echo "rc=$?" >> gpurun_out/t_cc.log
echo done
