#!/bin/bash
# round 2 (re-entry): where HEAD stands -- seam vs two-region x walls timing, bench, parity subset
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/m_smoke.txt 2>&1; echo smoke=$? >> gpurun_out/m_smoke.txt
for cfg in "" "WAVE25_SEAM=0"; do
  echo "== $cfg" >> gpurun_out/qt_m.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_m.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_m.txt 2>&1
  env $cfg timeout 300 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_m.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C2 stream 20 >> gpurun_out/qt_m.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/m_bench_c3.json 2> gpurun_out/m_bench_c3.err
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-probe > gpurun_out/m_bench_c2.json 2> gpurun_out/m_bench_c2.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_m.log 2>&1
echo "rc=$?" >> gpurun_out/t_m.log
echo done
