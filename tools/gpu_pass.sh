#!/bin/bash
# One GPU-box evidence pass (run from the repo root under gpurun):
#   bash tools/gpu_pass.sh TAG [tests] [bench] [shard] [nyt] [ncu] [ncu_nyt]
# Writes gpurun_out/TAG_*; copy the summaries worth keeping into profiles/.
set -u
tag=$1; shift
o=gpurun_out
mkdir -p $o
want() { [[ " $STEPS " == *" $1 "* ]]; }
STEPS=" $* "
summ() {
  python - "$1" <<'PY'
import json, sys
line = [l for l in open(sys.argv[1]) if l.startswith("{")]
if not line:
    print(sys.argv[1], "NO JSON"); sys.exit()
d = json.loads(line[-1])
r = d.get("roofline") or {}
e = d.get("e2e") or {}
ks = d.get("kernels") or {}
print(sys.argv[1].split("/")[-1], f"{d['value']/1e9:.3f} G ms/step={d['ms_per_step']:.2f}", f"K1frac={r.get('frac', 0):.3f}",
      f"e2e={(e or {}).get('value', 0)/1e9:.3f} G", {k: round(v, 3) for k, v in (d.get("kernel_ms") or {}).items()},
      {k: (round(v.get("ms", 0), 3), round(v.get("frac", 0), 3)) for k, v in ks.items() if isinstance(v, dict) and "frac" in v},
      "k5", (d.get("conservation") or {}).get("ms"),
      "cpu", (d.get("cpu_baseline") or {}).get("value"), d.get("clocks", {}).get("reasons"))
PY
}
if want tests; then
  python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $o/${tag}_smoke.log)"
  timeout 1500 python -m pytest tests -m gpu -q -x > $o/${tag}_gputests.log 2>&1; echo "gpu tests: $(tail -3 $o/${tag}_gputests.log)"
fi
if want bench; then
  t0=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 > $o/${tag}_bench_pm.json 2> $o/${tag}_bench_pm.err
  echo "default bench wall: $(( $(date +%s) - t0 )) s"; summ $o/${tag}_bench_pm.json
  t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err
  echo "reference arm wall: $(( $(date +%s) - t0 )) s"; tail -c 600 $o/${tag}_bench_ref.json
fi
if want shard; then
  timeout 900 python bench.py --shard 0/8 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > $o/${tag}_bench_shard0of8.json 2> $o/${tag}_bench_shard0of8.err
  summ $o/${tag}_bench_shard0of8.json
fi
if want nyt; then
  timeout 900 python bench.py --workload nytimes --no-cpu-baseline --steps 20 --warmup 5 > $o/${tag}_bench_nyt.json 2> $o/${tag}_bench_nyt.err
  summ $o/${tag}_bench_nyt.json
fi
if want api; then
  timeout 900 python tools/api_e2e.py --tag ${tag} --out-dir $o > $o/${tag}_api.log 2>&1; echo "api e2e rc=$? $(tail -c 400 $o/${tag}_api.log)"
fi
if want traj; then
  timeout 3000 python tools/trajectory.py --workload nytimes --gpu-iters 100 --cpu-iters 30 --cpu-seeds 1001,2002,3003 \
    --tag ${tag} --out-dir $o > $o/${tag}_traj.log 2>&1; echo "trajectory rc=$? $(tail -c 600 $o/${tag}_traj.log)"
fi
if want ncu; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"sample_kernel|phi_rebuild|theta_rebuild|prepare_kernel|context_kernel|ll_reduce" -s 6 -c 36 --csv \
    --log-file $o/${tag}_launches_pm.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "launch list rc=$?"
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel|theta_rebuild|phi_rebuild" -s 9 -c 3 \
    -o $o/${tag}_pm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $o/${tag}_ncu_pm.log 2>&1
  echo "pubmed capture rc=$?"
fi
if want ncu_nyt; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel" -s 3 -c 1 \
    -o $o/${tag}_k1_nyt python bench.py --workload nytimes --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "k1 nyt capture rc=$?"
fi
