#!/bin/bash
# round-2 end evidence: smoke, bench lines (C3, C2, fp64, 2-rank gloo with parity, reference arm),
# ncu launch list of the bench command, ncu --set full of the three fp32 kernels (traffic)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin_smoke.txt 2>&1; echo smoke=$? >> gpurun_out/fin_smoke.txt
timeout 900 python bench.py > gpurun_out/fin_bench_c3.json 2> gpurun_out/fin_bench_c3.err
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-probe > gpurun_out/fin_bench_c2.json 2> gpurun_out/fin_bench_c2.err
timeout 900 python bench.py --precision fp64 --no-cpu-baseline --no-probe > gpurun_out/fin_bench_fp64.json 2> gpurun_out/fin_bench_fp64.err
WAVE25_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --repeats 1 > gpurun_out/fin_bench_2rank.json 2> gpurun_out/fin_bench_2rank.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/fin_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > gpurun_out/fin_ncu_launches.log 2>&1
timeout 300 python scripts/prof_kinds.py C3 stream 1 > gpurun_out/fin_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_stream<\(int\)(248|24|128),' -s 3 -c 3 -o gpurun_out/fin_prof python scripts/prof_kinds.py C3 stream 1 > gpurun_out/fin_ncu_full.log 2>&1
echo done
