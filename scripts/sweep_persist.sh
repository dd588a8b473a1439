#!/bin/bash
for pe in 1 0; do for fk in 1 0; do for cz in 0 64 128; do
  E="WAVE25_PERSIST=$pe WAVE25_FORK=$fk"; [ $cz -gt 0 ] && E="$E WAVE25_CZ=$cz"
  env $E timeout 300 python scripts/quick_time.py C3 stream 60 2>&1 | sed "s/^/persist=$pe fork=$fk cz=$cz /" | tail -1
done; done; done
