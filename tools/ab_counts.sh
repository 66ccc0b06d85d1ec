#!/bin/bash
# A/B of the count kernels (K2 / K3 alone, K5) on the PubMed-shaped bench:
#   bash tools/ab_counts.sh TAG "ENV1" "ENV2" ...
tag=$1; shift
o=gpurun_out; mkdir -p $o
for envs in "$@"; do
  env $envs timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $o/${tag}_ab.json 2>/dev/null
  python - "$envs" $o/${tag}_ab.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[2]) if l.startswith("{")][-1])
k = d["kernels"]
print(f"{sys.argv[1]:24s} step {d['ms_per_step']:.2f} K1 {d['kernel_ms']['sample']:.2f} K2 {k['phi_rebuild']['ms']:.3f} "
      f"K3 {k['theta_rebuild']['ms']:.3f} inK2 {k['in_step_ms']['phi_rebuild']:.3f} inK3 {k['in_step_ms']['theta_rebuild']:.3f} "
      f"K5 {d['conservation']['ms']:.3f} ok={d['conservation']['ok']}")
PY
done
