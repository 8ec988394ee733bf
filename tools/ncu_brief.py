"""Print the headline metrics of an ncu report: python tools/ncu_brief.py rep.ncu-rep [kernel-substr]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if len(sys.argv) > 2 and sys.argv[2] not in name:
        continue
    print("==", name[:90])
    for w in want:
        if w in hdr:
            print(f"  {w} = {r[hdr.index(w)]} {units[hdr.index(w)]}")
    st = []
    for h, v in zip(hdr, r):
        if "smsp__average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("  stalls:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
