# wall scheduling knobs on top of the 40-plane wall chunks; fp64 wall chunk length
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out; out=gpurun_out/wallsched.txt; : > $out
for r in 1 2; do
for kv in "X=0" "WAVE25_WALL_PRIO=0" "WAVE25_SIDE2=1" "WAVE25_WALLS_LAST=1"; do echo "== C3 $kv" >> $out; env $kv timeout 300 python scripts/quick_time.py C3 stream 100 >> $out 2>&1; done
for cz in 0 40 24; do echo "== C3fp64 WALL_CZ=$cz" >> $out; WAVE25_WALL_CZ=$cz timeout 300 python scripts/quick_time.py C3 stream 60 fp64 >> $out 2>&1; done
for kv in "X=0" "WAVE25_WALL_PRIO=0" "WAVE25_SIDE2=1"; do echo "== C2 $kv" >> $out; env $kv timeout 300 python scripts/quick_time.py C2 stream 200 >> $out 2>&1; done
done
cat $out
