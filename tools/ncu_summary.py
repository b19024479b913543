"""Summarise an ncu --set full report: headline metrics, top stall reasons and the
hottest source lines (instructions / stall samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'lts__t_sector_hit_rate.pct',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'launch__shared_mem_per_block_dynamic', 'launch__block_size', 'launch__grid_size']
for r in rows[2:]:
    d = dict(zip(h, r))
    print("kernel:", d['Kernel Name'][:100])
    for k in KEYS:
        if k in d:
            print(f"  {k:70s} {d[k]}")
    st = [(k, d[k]) for k in h if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued')]
    st = sorted(st, key=lambda x: -float(x[1] or 0))[:10]
    for k, v in st:
        print('  stall', k[33:], v)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(rows) if 'Warp Stall Sampling (All Samples)' in r)
h = rows[hi]
si, ii = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
out = []
for r in rows[hi + 1:]:
    if r and r[0] != '':
        try:
            out.append((int(r[0]), r[1][:80], int(r[si] or 0), int(r[ii] or 0)))
        except ValueError:
            pass
ts, ti = max(1, sum(o[2] for o in out)), max(1, sum(o[3] for o in out))
print(f"source lines: {ts} stall samples, {ti} warp instructions")
for o in sorted(out, key=lambda x: -x[2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{o[0]:5d} {o[2] * 100 / ts:5.1f}% stall {o[3] * 100 / ti:5.1f}% inst  {o[1]}")
