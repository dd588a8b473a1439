set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python scripts/prof_kinds.py C3 stream 8
timeout 120 python scripts/prof_kinds.py C3 tb2 8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tb2 -c 1 -o gpurun_out/tb2_full python scripts/quick_time.py C3 tb2 4 > /dev/null 2>&1; echo ncu=$?
