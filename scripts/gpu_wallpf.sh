# wall-kernel L2 prefetch distance x x-wall tile variant (DESIGN.md §5 ablation)
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
out=gpurun_out/wallpf.txt; : > $out
for t in x24c16x128x1r x24c16x32x1 x24c16x32x1m4 x28c16x32x1m3 x24c16x64x1; do
 for pf in 1 3 6; do
  echo "== WALLX_TILE=$t WALL_PF=$pf" >> $out
  WAVE25_WALLX_TILE=$t WAVE25_WALL_PF=$pf timeout 300 python scripts/quick_time.py C3 stream 60 >> $out 2>&1
  WAVE25_WALLX_TILE=$t WAVE25_WALL_PF=$pf timeout 300 python scripts/prof_kinds.py C3 stream 6 >> $out 2>&1
 done
done
for pf in 0 2 4; do echo "== default WALL_PF=$pf" >> $out; WAVE25_WALL_PF=$pf timeout 300 python scripts/quick_time.py C3 stream 60 >> $out 2>&1; WAVE25_WALL_PF=$pf timeout 300 python scripts/prof_kinds.py C3 stream 6 >> $out 2>&1; done
cat $out
