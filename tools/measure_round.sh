#!/bin/bash
# One GPU-box pass that regenerates the judged evidence for a round (run from
# the repo root under gpurun):  bash tools/measure_round.sh r1g
# Writes gpurun_out/<tag>_*; copy the summaries worth keeping into profiles/.
set -u
tag=${1:-rX}
o=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $o/${tag}_smoke.log)"
timeout 1200 python -m pytest tests -m gpu -q > $o/${tag}_gputests.log 2>&1; echo "gpu tests: $(tail -1 $o/${tag}_gputests.log)"
# bench lines: the default command, the other workloads, the K sweep, the reference arm
t0=$(date +%s); timeout 900 python bench.py > $o/${tag}_bench_nyt.json 2> $o/${tag}_bench_nyt.err; echo "default bench wall: $(( $(date +%s) - t0 )) s"
timeout 900 python bench.py --workload pubmed > $o/${tag}_bench_pm.json 2> $o/${tag}_bench_pm.err
timeout 900 python bench.py --workload z4shard --no-cpu-baseline > $o/${tag}_bench_z4.json 2> $o/${tag}_bench_z4.err
for k in 128 256 4096; do
  timeout 600 python bench.py --topics $k --no-cpu-baseline --no-e2e > $o/${tag}_bench_k$k.json 2> $o/${tag}_bench_k$k.err
done
timeout 900 python bench.py --impl reference > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err
for f in $o/${tag}_bench_*.json; do
  python - "$f" <<'PY'
import json, sys
line = [l for l in open(sys.argv[1]) if l.startswith("{")]
if not line:
    print(sys.argv[1], "NO JSON"); sys.exit()
d = json.loads(line[-1])
r = d.get("roofline") or {}
e = d.get("e2e") or {}
print(sys.argv[1].split("/")[-1], f"{d['value']/1e9:.3f} G", f"frac={r.get('frac', 0):.3f}",
      f"e2e={e.get('value', 0)/1e9:.3f} G", d.get("kernel_ms"), d.get("clocks", {}).get("reasons"))
PY
done
# launch list of the default command (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sample_kernel|phi_rebuild|theta_rebuild|prepare_kernel|context_kernel|ll_reduce" -s 6 -c 36 --csv \
  --log-file $o/${tag}_launches_nyt.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "launch list rc=$?"
# full capture of K1 (iteration 3 of the default workload)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel" -s 3 -c 1 \
  -o $o/${tag}_k1_nyt python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "k1 capture rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel|theta_rebuild|phi_rebuild" -s 9 -c 3 \
  -o $o/${tag}_pm python bench.py --workload pubmed --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "pubmed capture rc=$?"
# loglik vs time, GPU against the oracle
timeout 1200 python tools/trajectory.py --workload nytimes --tag $tag --out-dir gpurun_out > $o/${tag}_traj.log 2>&1; echo "trajectory rc=$? $(tail -2 $o/${tag}_traj.log)"
bash tools/sanitize.sh
