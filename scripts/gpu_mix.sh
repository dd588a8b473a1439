# k_mix (interior + x walls in one grid) vs separate launches: timing
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for sc in C3 C2; do for m in 0 1 2 0 2; do WAVE25_MIX=$m timeout 300 python scripts/quick_time.py $sc stream 100 | sed "s/^/mix=$m /"; done; done > gpurun_out/mix_time2.txt 2>&1
WAVE25_MIX=2 WAVE25_WALL_PRIO=0 timeout 300 python scripts/quick_time.py C3 stream 100 | sed "s/^/mix=2 prio0 /" >> gpurun_out/mix_time2.txt
cat gpurun_out/mix_time2.txt
