#!/bin/bash
# round 2: default back to two-region x walls; fp64 bench; ncu --set full (source) of the 3 fp32 kernels
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1
timeout 300 python scripts/quick_time.py C3 stream 200 > gpurun_out/qt_n.txt 2>&1
timeout 300 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_n.txt 2>&1
timeout 300 python scripts/quick_time.py C3 stream 50 fp64 >> gpurun_out/qt_n.txt 2>&1
timeout 300 python scripts/prof_kinds.py C3 stream 10 fp64 >> gpurun_out/qt_n.txt 2>&1
timeout 900 python bench.py --precision fp64 --no-cpu-baseline --no-probe --steps 100 > gpurun_out/n_bench_fp64.json 2> gpurun_out/n_bench_fp64.err
timeout 300 python scripts/prof_kinds.py C3 stream 1 > gpurun_out/n_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_stream<\(int\)(248|24|128),' -s 3 -c 3 -o gpurun_out/prof_n python scripts/prof_kinds.py C3 stream 1 > gpurun_out/ncu_n.log 2>&1
echo done
