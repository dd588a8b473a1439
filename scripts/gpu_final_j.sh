# Round-end evidence refresh (development aid): smoke, full -m gpu suite, bench lines, ncu launch list,
# one ncu --set full capture of the interior kernel
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_j.txt 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gpu_tests_j.txt; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; echo bench=$?
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-probe > gpurun_out/bench_c2_j.json 2>/dev/null; echo c2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_j.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/ncu_bench_j.log 2>&1; echo ncul=$?
timeout 900 ncu --kernel-name-base demangled --set full --clock-control none --import-source on -k "regex:k_stream<\(int\)248, \(int\)248, \(int\)8, \(int\)1, \(int\)0" -s 2 -c 1 -o gpurun_out/interior_full_j python scripts/quick_time.py C3 stream 2 > gpurun_out/ncu_full_j.log 2>&1; echo ncuf=$?
cat gpurun_out/gpu_tests_j.txt
