#!/bin/bash
python -c "import torch; p=torch.cuda.get_device_properties(0); print('persist max', p.persisting_l2_cache_max_size if hasattr(p,'persisting_l2_cache_max_size') else '?')"
for cfg in "0 1" "64 1" "96 1" "96 0.5" "32 1"; do set -- $cfg
  WAVE25_L2MB=$1 WAVE25_L2HR=$2 timeout 300 python scripts/quick_time.py C3 stream 40 2>&1 | sed "s/^/l2mb=$1 hr=$2 /" | tail -1
done
