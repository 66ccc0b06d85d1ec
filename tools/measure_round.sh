#!/bin/bash
# One GPU-box pass that regenerates the judged evidence for a round (run from
# the repo root under gpurun):  bash tools/measure_round.sh r2
# Writes gpurun_out/<tag>_*; tools/collect_round.py <tag> copies the summaries
# into profiles/.  (The NYTimes loglik trajectory with its oracle seed band is
# a separate, longer pass: bash tools/gpu_pass.sh <tag> traj.)
set -u
tag=${1:-rX}
o=gpurun_out
mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $o/${tag}_smoke.log)"
timeout 1500 python -m pytest tests -m gpu -q > $o/${tag}_gputests.log 2>&1; echo "gpu tests: $(tail -1 $o/${tag}_gputests.log)"
# bench lines: the default command (PubMed-shape), the reference arm, the
# 8-way shard proxy, the other BASELINE configs, the K sweep
t0=$(date +%s); timeout 900 python bench.py > $o/${tag}_bench_pm.json 2> $o/${tag}_bench_pm.err; echo "default bench wall: $(( $(date +%s) - t0 )) s"
timeout 900 python bench.py --impl reference > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err
timeout 900 python bench.py --shard 0/8 --no-cpu-baseline --no-e2e > $o/${tag}_bench_shard0of8.json 2> $o/${tag}_bench_shard0of8.err
timeout 900 python bench.py --shard 7/8 --no-cpu-baseline --no-e2e > $o/${tag}_bench_shard7of8.json 2> $o/${tag}_bench_shard7of8.err
timeout 900 python bench.py --workload nytimes --no-cpu-baseline > $o/${tag}_bench_nyt.json 2> $o/${tag}_bench_nyt.err
timeout 900 python bench.py --workload z4shard --no-cpu-baseline > $o/${tag}_bench_z4.json 2> $o/${tag}_bench_z4.err
for k in 128 256 4096; do
  timeout 600 python bench.py --workload nytimes --topics $k --no-cpu-baseline --no-e2e > $o/${tag}_bench_k$k.json 2> $o/${tag}_bench_k$k.err
done
timeout 900 python tools/api_e2e.py --tag ${tag} --out-dir $o > $o/${tag}_api.log 2>&1; echo "api e2e rc=$?"
for f in $o/${tag}_bench_*.json; do
  python - "$f" <<'PY'
import json, sys
line = [l for l in open(sys.argv[1]) if l.startswith("{")]
if not line:
    print(sys.argv[1], "NO JSON"); sys.exit()
d = json.loads(line[-1])
r = d.get("roofline") or {}
e = d.get("e2e") or {}
print(sys.argv[1].split("/")[-1], f"{d['value']/1e9:.3f} G", f"ms={d['ms_per_step']:.2f}", f"frac={r.get('frac', 0):.3f}",
      f"e2e={(e or {}).get('value', 0)/1e9:.3f} G", d.get("kernel_ms"), d.get("clocks", {}).get("reasons"))
PY
done
# launch list of the default command (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sample_kernel|phi_rebuild|theta_rebuild|prepare_kernel|context_kernel|ll_reduce" -s 6 -c 36 --csv \
  --log-file $o/${tag}_launches_pm.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "launch list rc=$?"
# full captures at ITERATION 6 (inside bench.py's default timed range,
# iterations 3..12): K1 / K2 / K3 of the default workload, K5, K1 on
# NYTimes-shape.  Matched launches: K2, K3 (initial counts), then per
# iteration K1, K3, K2 -- so -s 20 is iteration 6 (--warmup 5).
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel|theta_rebuild|phi_rebuild" -s 20 -c 3 \
  -o $o/${tag}_pm python bench.py --steps 2 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "pubmed capture rc=$?"
# K3 alone (in the combined capture above, K3 -- launched on the side stream
# beside K2 -- comes back with most metric passes NaN)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"theta_rebuild" -s 6 -c 1 \
  -o $o/${tag}_k3_pm python bench.py --steps 2 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "k3 capture rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k5_" -c 6 \
  -o $o/${tag}_k5_pm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "k5 capture rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel" -s 6 -c 1 \
  -o $o/${tag}_k1_nyt python bench.py --workload nytimes --steps 2 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "k1 nyt capture rc=$?"
if [ "${SANITIZE:-1}" = 1 ]; then bash tools/sanitize.sh; fi
