#!/bin/bash
# round 2: cluster-multicast interior variants (rc2, rc4): bitwise, timing, DRAM bytes
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants_bitwise and rc" -p no:cacheprovider > gpurun_out/t_variants.log 2>&1
echo "rc=$?" >> gpurun_out/t_variants.log
for t in 248x8x1r 248x8x1rc2 248x8x1rc4; do
  for c in C3 C2; do
    WAVE25_INNER_TILE=$t timeout 300 python scripts/quick_time.py $c stream 100 >> gpurun_out/qt_$t.txt 2>&1
    WAVE25_INNER_TILE=$t timeout 300 python scripts/prof_kinds.py $c stream 10 >> gpurun_out/qt_$t.txt 2>&1
  done
done
for t in 248x8x1r 248x8x1rc2; do
  WAVE25_INNER_TILE=$t timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_stream -s 6 -c 6 --csv python scripts/prof_kinds.py C3 stream 2 > gpurun_out/ncu_$t.csv 2>&1
done
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_peer.log 2>&1
echo "rc=$?" >> gpurun_out/t_peer.log
echo done
