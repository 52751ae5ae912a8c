"""Summarise an ncu report: key throughput metrics + warp stall breakdown."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
for k in want:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {vals[i]:>18s} {units[i]}")
print("--- stall reasons (warp cycles per issued instruction) ---")
stalls = []
for i, k in enumerate(h):
    if k.startswith("smsp__average_warp_latency_issue_stalled_") or k.startswith("smsp__average_warps_issue_stalled_"):
        if k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), k))
            except ValueError:
                pass
for v, k in sorted(stalls, reverse=True)[:14]:
    print(f"{v:8.3f}  {k}")
