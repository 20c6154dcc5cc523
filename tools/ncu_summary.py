"""Summarise an .ncu-rep: key SOL/occupancy/stall metrics (raw page)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, vals = rows[0], rows[1], rows[2:]
want = sys.argv[2:] or ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__inst_executed.sum", "smsp__inst_executed.avg.per_cycle_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "sm__maximum_warps_per_active_cycle_pct", "achieved_occupancy"]
for v in vals:
    for w in want:
        for i, k in enumerate(h):
            if k == w or (w.endswith("*") and k.startswith(w[:-1])):
                print("%-70s %s %s" % (k, v[i], units[i]))
