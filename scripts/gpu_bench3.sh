python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
timeout 600 python bench.py --precision fp64 --no-cpu-baseline --no-probe > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err; echo b64=$?; cat gpurun_out/bench_fp64.json
timeout 600 python bench.py --kernel tb2 --no-cpu-baseline --no-probe --no-e2e > gpurun_out/bench_tb2.json 2> gpurun_out/bench_tb2.err; echo btb2=$?; cat gpurun_out/bench_tb2.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo bref=$?; cat gpurun_out/bench_ref.json
