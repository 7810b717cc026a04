"""Summarise an ncu --set full report: per kernel duration, DRAM traffic,
occupancy, pipes, top warp stall reasons.  usage: python tools/ncu_summary.py REP.ncu-rep"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "launch__occupancy_limit_registers",
     "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for row in rows[2:]:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    print(f"== {d['Kernel Name'][:90]}")
    for k in M:
        if k in d:
            print(f"   {k:62s} {d[k]:>14s} {u.get(k, '')}")
    stalls = [(k, float(d[k])) for k in hdr
              if k.startswith("smsp__average_warp_latency_issue_stalled_")
              and k.endswith(".ratio") and d[k] not in ("", "n/a")]
    if not stalls:
        stalls = [(k, float(d[k].replace(",", ""))) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and d[k] not in ("", "n/a")
                  and not k.endswith("not_issued")]
    tot = sum(v for _, v in stalls) or 1.0
    for k, v in sorted(stalls, key=lambda kv: -kv[1])[:6]:
        print(f"   stall {k.split('stalled_')[-1]:55s} {v / tot:6.1%}")
