for t in y64x8x1m3 y248x8x1r y128x8x1m3 y128x8x1; do echo "ytile=$t"; WAVE25_WALLY_TILE=$t timeout 120 python scripts/prof_kinds.py C3 stream 6 | grep -E "walls|total"; done
for t in x24c16x32x1 x24c16x32x1m3 x32c16x32x1 x24c16x64x1; do echo "xtile=$t"; WAVE25_WALLX_TILE=$t timeout 120 python scripts/prof_kinds.py C3 stream 6 | grep -E "xwalls"; done
timeout 120 python scripts/quick_time.py C3 stream 50
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py 2>&1 | tail -3
