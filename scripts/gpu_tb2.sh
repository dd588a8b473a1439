set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_tb2.py -x -q -k "C1-2 or RAGGED" 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_tb2.py -q 2>&1 | tail -15
timeout 120 python scripts/quick_time.py C3 stream 50
timeout 120 python scripts/quick_time.py C3 tb2 50
WAVE25_T2_TILE=56x16 timeout 120 python scripts/quick_time.py C3 tb2 50
