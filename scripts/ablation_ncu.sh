M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sector_hit_rate.pct
for sh in default gmem_32x4x1 gmem_8x8x8 smem_u st_smem_32x16 st_reg_shft_32x16 st_reg_fixed_32x16 st_reg_fixed_32x32 semi_32x16; do
  if [ $sh = default ]; then E=""; K='regex:k_stream<\(int\)248'; else E="WAVE25_ABLATION=$sh"; K='regex:w25::(k_gmem<|k_st<|k_smem_u|k_semi<)'; fi
  env $E timeout 600 ncu --kernel-name-base demangled --metrics $M --clock-control none -k "$K" -c 1 --csv python scripts/quick_time.py C3 stream 2 2>/dev/null | grep -v "^==" > gpurun_out/abl_$sh.csv
  head -c 300 gpurun_out/abl_$sh.csv; echo
done
