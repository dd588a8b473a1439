# Round evidence: ncu full capture of the default kernels, launch list, bench lines
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -c 3 -o gpurun_out/stream_full python scripts/quick_time.py C3 stream 2 > /dev/null 2>&1; echo ncu=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/ncu_bench.log 2>&1; echo ncul=$?
timeout 600 python bench.py --precision fp64 --no-cpu-baseline --no-probe > gpurun_out/bench_fp64.json 2>/dev/null; echo b64=$?
