#!/bin/bash
# round 2: bench line with per-kind roofline fractions (C3 default run, driver-style)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/gg_build.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/gg_bench_c3.json 2> gpurun_out/gg_bench_c3.err
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-probe > gpurun_out/gg_bench_c2.json 2> gpurun_out/gg_bench_c2.err
echo done
