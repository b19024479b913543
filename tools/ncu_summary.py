"""Summarise an ncu --set full report (raw page) for the kernel: key metrics + top stalls."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print("kernel:", d.get("Kernel Name", "")[:90])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]:>16s} {u[k]}")
    stalls = []
    for k, v in d.items():
        if k.startswith("smsp__average_warp_latency_issue_stalled") or (k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")):
            try:
                stalls.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
    for v, k in sorted(stalls, reverse=True)[:12]:
        print(f"  stall {k:70s} {v:12.1f}")
