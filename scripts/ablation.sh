# Code-shape ablation on C3: device time of the interior launch
# per shape (CUDA events, prof_kinds) and ncu counters of one launch.
python -c "import __graft_entry__ as g; g.build()" || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sector_hit_rate.pct
for sh in default gmem_32x4x1 gmem_8x8x8 smem_u st_smem_32x16 st_reg_shft_32x16 st_reg_fixed_32x16 st_reg_fixed_32x32; do
  if [ $sh = default ]; then E=""; K='regex:k_stream<248'; else E="WAVE25_ABLATION=$sh"; K='regex:k_gmem|k_smem_u|k_st<'; fi
  echo "== $sh"; env $E timeout 300 python scripts/prof_kinds.py C3 stream 4 | grep interior
  env $E timeout 600 ncu --metrics $M --clock-control none -k "$K" -c 1 --csv python scripts/quick_time.py C3 stream 2 2>/dev/null | grep -v "^==" | tail -n +2 > gpurun_out/abl_$sh.csv
done
