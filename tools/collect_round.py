"""Copy a measure_round.sh pass (gpurun_out/<tag>_*) into profiles/: bench
lines, ncu summaries, the launch-list summary, the loglik trajectory and the
sanitizer tails.  Usage: python tools/collect_round.py r1i"""
import csv
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")

for w in ["pm", "ref", "shard0of8", "shard7of8", "nyt", "z4", "k128", "k256", "k4096"]:
    src = os.path.join(O, f"{tag}_bench_{w}.json")
    lines = [l for l in open(src) if l.startswith("{")] if os.path.exists(src) else []
    if lines:
        open(os.path.join(P, f"{tag}_bench_{w}.json"), "w").write(lines[-1])
summ = os.path.join(P, "ncu_summary.py")
for rep, out, top in [(f"{tag}_k1_nyt.ncu-rep", f"{tag}_nyt_sample_kernel_ncu.txt", "30"),
                      (f"{tag}_pm.ncu-rep", f"{tag}_pubmed_k1_k2_k3_ncu.txt", "25"),
                      (f"{tag}_k3_pm.ncu-rep", f"{tag}_pubmed_k3_ncu.txt", "20"),
                      (f"{tag}_k5_pm.ncu-rep", f"{tag}_pubmed_k5_ncu.txt", "15")]:
    if os.path.exists(os.path.join(O, rep)):
        with open(os.path.join(P, out), "w") as fh:
            subprocess.run([sys.executable, summ, os.path.join(O, rep), top], stdout=fh, stderr=subprocess.STDOUT)
lst = os.path.join(O, f"{tag}_launches_pm.csv")
if os.path.exists(lst):
    shutil.copy(lst, P)
    rows = [r for r in csv.reader(open(lst)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tm = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    L = {}
    for r in rows[1:]:
        d = L.setdefault(int(r[ii]), {"k": r[ki].split("(")[0]})
        v, u = float(r[vi].replace(",", "")), r[ui]
        if r[mi] == "gpu__time_duration.sum":
            d["ms"] = v * tm.get(u, 1e-6)
        elif r[mi].startswith("dram__bytes_read"):
            d["rd"] = v * sc[u] / 1e9
        elif r[mi].startswith("dram__bytes_write"):
            d["wr"] = v * sc[u] / 1e9
    out = ["ncu launch list (iteration kernels only): python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e",
           "(PubMed-shape, K=1024, 1 B200: the bench default), launches 6..41; per-launch times are cold-cache and serialised",
           "(compare shares, not absolutes); bench.py runs K3 on a side stream beside K2, ncu serialises them", "",
           f"{'id':>3} {'kernel':42s} {'ms':>8} {'dram_read_GB':>12} {'dram_write_GB':>13}"]
    tot = {}
    for i in sorted(L):
        d = L[i]
        out.append(f"{i:3d} {d['k'][:42]:42s} {d.get('ms', 0):8.3f} {d.get('rd', 0):12.3f} {d.get('wr', 0):13.3f}")
        tot[d["k"]] = tot.get(d["k"], 0) + d.get("ms", 0)
    s = sum(tot.values()) or 1.0
    out += ["", "share of serialised kernel time:"]
    out += [f"  {k[:42]:42s} {100 * v / s:6.2f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    open(os.path.join(P, f"{tag}_launch_summary.txt"), "w").write("\n".join(out) + "\n")
for ext in ("csv", "json"):
    f = os.path.join(O, f"{tag}_loglik_nytimes.{ext}")
    if os.path.exists(f):
        shutil.copy(f, P)
with open(os.path.join(P, f"{tag}_sanitizer.txt"), "w") as fh:
    for t in ["memcheck", "racecheck", "synccheck", "initcheck", "memcheck_tests", "memcheck_k23", "memcheck_phases"]:
        f = os.path.join(O, f"san_{t}.log")
        if os.path.exists(f):
            fh.write(f"== {t}\n" + "".join(open(f).readlines()[-3:]))
print("collected", tag)

# roofline.traffic lookup for bench.py: DRAM bytes of the captured K1 launch
# (iteration 6, inside the default timed range) per workload
import io
import json


def k1_dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:sample_kernel"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    h, u, v = rows[0], rows[1], rows[2]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    get = lambda m: float(v[h.index(m)].replace(",", "")) * sc.get(u[h.index(m)], 1)
    return {"kernel": v[h.index("Kernel Name")].split("(")[0], "dram_read_bytes": int(get("dram__bytes_read.sum")),
            "dram_write_bytes": int(get("dram__bytes_write.sum")),
            "bytes_per_launch": int(get("dram__bytes_read.sum") + get("dram__bytes_write.sum")),
            "lts_hit_rate_pct": float(v[h.index("lts__t_sector_hit_rate.pct")])}


tf = os.path.join(P, "sample_kernel_traffic.json")
traffic = json.load(open(tf)) if os.path.exists(tf) else {}
for key, rep, what in [("pubmed-1024", f"{tag}_pm.ncu-rep", "bench.py --steps 2 --warmup 5 (default workload)"),
                       ("nytimes-1024", f"{tag}_k1_nyt.ncu-rep", "bench.py --workload nytimes --steps 2 --warmup 5")]:
    r = os.path.join(O, rep)
    if os.path.exists(r):
        d = k1_dram(r)
        if d:
            d["source"] = f"profiles/{tag}_* (ncu --set full of `{what}`, the K1 launch of iteration 6)"
            d["iteration"] = 6
            traffic[key] = d
traffic["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch (ncu --set full at iteration 6, "
                   "inside bench.py's default timed range of iterations 3..12); bench.py reports the entry matching its "
                   "--workload and K as roofline.traffic.  Algorithmic bytes per launch are reported live by bench.py.")
json.dump(traffic, open(tf, "w"), indent=2)
print("traffic entries", sorted(k for k in traffic if k != "note"))
