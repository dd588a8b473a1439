python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -c 3 -o gpurun_out/stream_full python scripts/quick_time.py C3 stream 2 > /dev/null 2>&1; echo ncu=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/ncu_bench.log 2>&1; echo ncul=$?
