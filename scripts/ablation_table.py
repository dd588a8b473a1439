"""Summarise the code-shape ablation ncu CSVs (scripts/ablation_ncu.sh) into a table."""
import csv, sys
order = ["default", "gmem_32x4x1", "gmem_8x8x8", "smem_u", "st_smem_32x16", "st_reg_shft_32x16",
         "st_reg_fixed_32x16", "st_reg_fixed_32x32", "semi_32x16"]
pts = 1007681536
d0 = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
print(f"{'shape':22s} {'ms(ncu)':>8s} {'DRAM B/pt':>9s} {'inst/pt':>8s} {'regs':>5s} {'warps%':>7s} {'issue%':>7s} {'smem wf/pt':>10s} {'L2hit%':>7s}")
for sh in order:
    rows = [r for r in csv.reader(open(f"{d0}/abl_{sh}.csv")) if len(r) > 14]
    hdr = rows[0]
    ki, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    d = {r[ki]: (float(r[vi].replace(",", "")), r[ui]) for r in rows[1:]}
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3,
          "msecond": 1.0, "nsecond": 1e-6}
    g = lambda k: d[k][0] * sc.get(d[k][1], 1.0)
    b = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
    print(f"{sh:22s} {g('gpu__time_duration.sum'):8.3f} {b / pts:9.2f} {d['smsp__inst_executed.sum'][0] * 32 / pts:8.1f} "
          f"{d['launch__registers_per_thread'][0]:5.0f} {d['sm__warps_active.avg.pct_of_peak_sustained_active'][0]:7.1f} "
          f"{d['smsp__issue_active.avg.pct_of_peak_sustained_active'][0]:7.1f} "
          f"{d['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'][0] / pts:10.2f} {d['lts__t_sector_hit_rate.pct'][0]:7.1f}")
