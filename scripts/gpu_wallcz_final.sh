# wall chunk cap (W25_WALL_CZ_MAX = 40): bench lines + parity subset
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_k.txt 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err; echo bench=$?
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-probe > gpurun_out/bench_c2_k.json 2>/dev/null; echo c2=$?
for k in stream tb2 pair; do timeout 300 python scripts/quick_time.py C3 $k 60; done > gpurun_out/kinds_k.txt 2>&1
timeout 300 python scripts/quick_time.py C3 stream 60 fp64 >> gpurun_out/kinds_k.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_k.txt; echo tests=$?
cat gpurun_out/kinds_k.txt gpurun_out/gpu_tests_k.txt
