# Round-end evidence (development aid): bench lines (C3 default, C2, fp64, pair), the ncu launch
# list of the default bench, one ncu --set full capture of the interior kernel, the C2 full-run
# parity number.
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-probe > gpurun_out/bench_c2.json 2>/dev/null; echo c2=$?
timeout 600 python bench.py --precision fp64 --no-cpu-baseline --no-probe > gpurun_out/bench_fp64.json 2>/dev/null; echo fp64=$?
timeout 600 python bench.py --kernel pair --no-cpu-baseline --no-probe > gpurun_out/bench_pair.json 2>/dev/null; echo pair=$?
timeout 600 python bench.py --kernel tb2 --no-cpu-baseline --no-probe > gpurun_out/bench_tb2.json 2>/dev/null; echo tb2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/ncu_bench.log 2>&1; echo ncul=$?
timeout 900 ncu --kernel-name-base demangled --set full --clock-control none --import-source on -k "regex:k_stream<\(int\)248, \(int\)248, \(int\)8, \(int\)1, \(int\)0" -s 2 -c 1 -o gpurun_out/interior_full python scripts/quick_time.py C3 stream 2 > gpurun_out/ncu_full.log 2>&1; echo ncuf=$?
timeout 900 python -m pytest -q -s tests/test_gpu_parity.py -k c2_full 2>&1 | grep -E "C2 500|passed|failed" > gpurun_out/c2_full.txt; cat gpurun_out/c2_full.txt
