"""Summarise an ncu --set full report (here, no GPU): key counters + per-source-line stall samples."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25

def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
hdr, units, vals = raw[0], raw[1], raw[2]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__cluster_dim_x", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
out = {}
for h, u, v in zip(hdr, units, vals):
    if h in KEYS:
        out[h] = (v, u)
for k in KEYS:
    if k in out:
        print(f"{k:95s} {out[k][0]:>16s} {out[k][1]}")
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "cuda,sass"]))))
agg, cur = {}, None
for r in src:
    if len(r) < 5 or r[0] in ("File Path", "Function Name", "Line No"):
        continue
    if r[0]:
        cur = (r[0], r[1][:100])
        try:
            agg[cur] = int(r[4])
        except ValueError:
            agg[cur] = 0
tot = sum(agg.values()) or 1
print(f"--- stall samples by source line (total {tot})")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:9d} {100*v/tot:5.1f}%  L{k[0]:>4s}  {k[1]}")
