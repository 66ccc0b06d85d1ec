"""Summarise an ncu --set full report: headline metrics, stall reasons and the
hottest source lines (by instructions executed).  Usage:
    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__shared_mem_per_block_dynamic"]
print("== metrics")
for i, h in enumerate(hdr):
    if h in want:
        print(f"  {h} = {vals[i]} {units[i]}")
print("== stall reasons (pc samples)")
items = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            items.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in items) or 1
for v, h in sorted(items, reverse=True)[:10]:
    print(f"  {h:28s} {100 * v / tot:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
cur = None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            agg[(cur, int(r[0]))] = (int(r[7]), int(r[4]), r[1].strip()[:80])
        except ValueError:
            pass
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"== hottest source lines (total {ti / 1e9:.2f} G warp-instructions)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"  {k[0]}:{k[1]:<4d} inst {100 * v[0] / ti:5.1f}%  stall-samples {100 * v[1] / ts:5.1f}%  {v[2]}")
