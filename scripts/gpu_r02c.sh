#!/bin/bash
# round 2: origin shift + x-wall interleave A/B; cluster variant with CTA-scope arrives
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "" "WAVE25_NO_ORIGIN=1" "WAVE25_XINTER=0" "WAVE25_NO_ORIGIN=1 WAVE25_XINTER=0" "WAVE25_INNER_TILE=248x8x1rc2"; do
  echo "== $cfg" >> gpurun_out/qt_c.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 100 >> gpurun_out/qt_c.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_c.txt 2>&1
  env $cfg timeout 300 python scripts/quick_time.py C2 stream 200 >> gpurun_out/qt_c.txt 2>&1
done
for cfg in "" "WAVE25_NO_ORIGIN=1"; do
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_stream -s 6 -c 6 --csv python scripts/prof_kinds.py C3 stream 2 > gpurun_out/ncu_c_${cfg:-dflt}.csv 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_horizon.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_all.log 2>&1
echo "rc=$?" >> gpurun_out/t_all.log
echo done
