# TMA L2 promotion of the wall kernels' centre-only loads (64-B rows): timing + DRAM bytes
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
out=gpurun_out/wallpromo.txt; : > $out
for v in 2 0 1 2 0 1; do
  echo "== WALL_L2PROMO=$v" >> $out
  WAVE25_WALL_L2PROMO=$v timeout 300 python scripts/quick_time.py C3 stream 100 >> $out 2>&1
  WAVE25_WALL_L2PROMO=$v timeout 300 python scripts/prof_kinds.py C3 stream 6 >> $out 2>&1
done
for v in 2 0 1; do
  echo "== ncu WALL_L2PROMO=$v" >> $out
  WAVE25_WALL_L2PROMO=$v timeout 600 ncu --kernel-name-base demangled --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k "regex:k_stream<\(int\)(24|128), " -s 4 -c 4 python scripts/quick_time.py C3 stream 3 >> $out 2>&1
done
for v in 2 0 1; do echo "== C2 WALL_L2PROMO=$v" >> $out; WAVE25_WALL_L2PROMO=$v timeout 300 python scripts/quick_time.py C2 stream 200 >> $out 2>&1; done
grep -v "^==PROF==" $out | grep -E "==|ms/step|walls|dram|duration|hit_rate|k_stream"
