# round-end: smoke, full -m gpu suite, bench lines with y walls on their own side stream
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_l.txt 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; echo bench=$?
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-probe > gpurun_out/bench_c2_l.json 2>/dev/null; echo c2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_l.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/ncu_bench_l.log 2>&1; echo ncul=$?
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_l.txt; echo tests=$?
cat gpurun_out/gpu_tests_l.txt
