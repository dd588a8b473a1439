#!/bin/bash
for cz in ${CZS:-32 64 128 205 342 512 1024}; do WAVE25_CZ=$cz timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -k regex:k_stream -c 3 --csv --log-file gpurun_out/cz_$cz.csv python scripts/quick_time.py C3 stream 3 > /dev/null 2>&1; done
