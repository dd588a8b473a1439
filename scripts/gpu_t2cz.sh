for cz in 32 64 128 1024; do echo "cz=$cz"; WAVE25_T2_CZ=$cz timeout 120 python scripts/prof_kinds.py C3 tb2 4 | grep -E "interior"; done
