#!/bin/bash
# block order x L2 policy x prefetch (development aid)
SC=${1:-C3}
for o in ${ORDERS:-0 1 2 4}; do for up in ${UPOLS:-0 1}; do for pf in ${PFS:-2}; do for iv in ${INNER:-128x8x1}; do
  WAVE25_INNER_TILE=$iv WAVE25_PF=$pf WAVE25_ORDER=$o WAVE25_UPOL=$up timeout 300 python scripts/quick_time.py $SC stream 40 2>&1 | sed "s/^/$iv order=$o upol=$up pf=$pf /" | tail -1
done; done; done; done
