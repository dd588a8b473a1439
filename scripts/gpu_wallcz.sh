# wall chunk length (number of wall CTAs beside the interior), C3 and C2
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out; out=gpurun_out/wallcz2.txt; : > $out
for r in 1 2; do
for cz in 0 24 32 40 48 57 64 80; do echo "== C3 WALL_CZ=$cz" >> $out; WAVE25_WALL_CZ=$cz timeout 300 python scripts/quick_time.py C3 stream 100 >> $out 2>&1; done
for cz in 0 8 12 16 24 32 43; do echo "== C2 WALL_CZ=$cz" >> $out; WAVE25_WALL_CZ=$cz timeout 300 python scripts/quick_time.py C2 stream 200 >> $out 2>&1; done
done
WAVE25_WALL_CZ=57 timeout 300 python scripts/prof_kinds.py C3 stream 6 >> $out 2>&1
cat $out
