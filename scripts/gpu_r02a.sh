#!/bin/bash
# round 2, first GPU pass: new horizon + peer tests, quick bench N=1, 2-rank bench on one GPU (gloo)
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_horizon.py tests/test_gpu_peer.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/tests_new.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests_new.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "peer or slab" -p no:cacheprovider > gpurun_out/tests_peer_old.log 2>&1
echo "rc=$?" >> gpurun_out/tests_peer_old.log
timeout 600 python bench.py --steps 20 --warmup 3 --repeats 3 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err
WAVE25_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --repeats 1 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo done
