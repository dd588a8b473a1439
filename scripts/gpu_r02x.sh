#!/bin/bash
# round 2: compute-sanitizer, one tool per call: bash scripts/gpu_r02x.sh memcheck|racecheck|synccheck|initcheck
cd $GRAFT_REPO_ROOT
tool=${1:-memcheck}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1
timeout 600 python scripts/sanitize_run.py > gpurun_out/x_plain_$tool.log 2>&1 && \
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/x_$tool.log 2>&1
echo "rc=$?" >> gpurun_out/x_$tool.log
echo done
