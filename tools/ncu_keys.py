#!/usr/bin/env python3
"""Print the key metrics of an ncu raw-page CSV (ncu -i rep --page raw --csv): duration, DRAM bytes
and throughput, L1/L2 hit rates, occupancy, registers, issue activity and the top stall reasons."""
import csv
import io
import sys

rows = list(csv.reader(io.StringIO(open(sys.argv[1]).read())))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print(d.get("Kernel Name", "")[:90])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "lts__t_sectors.sum",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "launch__occupancy_limit_registers"]
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k]} {u.get(k, '')}")
    st = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled") or
          (k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"))]
    vals = []
    for k, v in st:
        try:
            vals.append((float(v.replace(",", "")), k))
        except ValueError:
            pass
    for v, k in sorted(vals, reverse=True)[:8]:
        print(f"  stall {k.split('stalled_')[-1]} = {v}")
