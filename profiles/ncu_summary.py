"""Summarise an ncu --set full report: headline metrics, stall reasons and the
hottest source lines (by instructions executed), for every kernel in the
report or only those matching a regex.  Usage:
    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [topN] [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilt = sys.argv[3] if len(sys.argv) > 3 else None

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sass__inst_executed_shared_loads"]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units = rows[0], rows[1]
kcol = hdr.index("Kernel Name")
seen = set()
for vals in rows[2:]:
    name = vals[kcol]
    if kfilt and not re.search(kfilt, name):
        continue
    short = name.split("(")[0]
    if short in seen:
        continue
    seen.add(short)
    print(f"#### {short}")
    print("== metrics")
    for i, h in enumerate(hdr):
        if h in WANT:
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
    esc = re.escape(short.split("<")[0].replace("void ", "").strip())
    src = ncu("--page", "source", "--csv", "--print-source=cuda,sass", "-k", f"regex:{esc}")
    agg = {}
    cur = None
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
            try:
                key = (cur, int(r[0]))
                old = agg.get(key, (0, 0, ""))
                agg[key] = (old[0] + int(r[7]), old[1] + int(r[4]), r[1].strip()[:80])
            except ValueError:
                pass
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"== hottest source lines (total {ti / 1e9:.2f} G warp-instructions)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"  {k[0]}:{k[1]:<4d} inst {100 * v[0] / ti:5.1f}%  stall-samples {100 * v[1] / ts:5.1f}%  {v[2]}")
    print()
