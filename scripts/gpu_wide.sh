for t in x24c16x32x1 x28c16x32x1 x28c16x64x1 x28c16x32x1m3; do echo "xtile=$t"; WAVE25_WALLX_TILE=$t timeout 120 python scripts/prof_kinds.py C3 stream 6 | grep -E "xwalls"; done
