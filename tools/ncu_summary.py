"""Compact summary of an ncu --set full report (one kernel): key metrics."""
import csv, io, subprocess, sys
rep = sys.argv[1]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
     "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
     "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
     "launch__block_size", "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
print("kernel:", vals[hdr.index("Kernel Name")][:90])
for m in M:
    if m in hdr:
        i = hdr.index(m)
        print(f"  {m:75s} {vals[i]:>14s} {units[i]}")
