#!/bin/bash
# round 2: bench at N>1 on one (time-shared) B200: 4 ranks weak (ranks 1, 2 with both neighbours
# mapped over IPC) and 2 ranks strong (C4 split) -- each line carries the bitwise parity bit
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bb_build.log 2>&1
WAVE25_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 6 --warmup 3 --repeats 1 --no-e2e > gpurun_out/bb_bench_4rank.json 2> gpurun_out/bb_bench_4rank.err
WAVE25_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --scaling strong --steps 10 --warmup 3 --repeats 1 > gpurun_out/bb_bench_2rank_strong.json 2> gpurun_out/bb_bench_2rank_strong.err
echo done
