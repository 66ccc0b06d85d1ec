"""Share of K1's instructions / stall samples by code region, from an
`ncu --set full --import-source on` report: python tools/probes/k1_regions.py rep"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", "regex:sample_kernel"],
                     capture_output=True, text=True).stdout
agg, cur = {}, None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            k = (cur, int(r[0])); o = agg.get(k, (0, 0)); agg[k] = (o[0] + int(r[7]), o[1] + int(r[4]))
        except ValueError:
            pass
ti = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
src = open("paper_1803_04631_b200/csrc/k_sample.cu").read().split("\n")
def find(p):
    return next(i + 1 for i, l in enumerate(src) if p in l)
def rng(a, b):
    i = sum(v[0] for k, v in agg.items() if k[0] == "k_sample.cu" and a <= k[1] <= b)
    s = sum(v[1] for k, v in agg.items() if k[0] == "k_sample.cu" and a <= k[1] <= b)
    return f"inst {100 * i / ti:5.1f}%  stalls {100 * s / ts:5.1f}%"
print("total G warp-inst", round(ti / 1e9, 2))
print("build_context  ", rng(find("__device__ __forceinline__ void build_context"), find("// One CTA per word that the schedule splits")))
print("first_above    ", rng(find("__device__ __forceinline__ uint32_t first_above"), find("__device__ __forceinline__ uint32_t first_above") + 6))
print("batch setup    ", rng(find("    while (true) {"), find("// ---- 1. entry-parallel pass")))
print("pass           ", rng(find("// ---- 1. entry-parallel pass"), find("// ---- 2. token-parallel draws")))
print("draws          ", rng(find("// ---- 2. token-parallel draws"), find("// log p(w|d) (L_d + K a) of the iteration-start model")))
print("epilogue       ", rng(find("// ---- deterministic reductions"), find("// ---- deterministic reductions") + 16))
