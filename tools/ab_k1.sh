#!/bin/bash
# A/B timing of the hot path under env-var tuning knobs (GPU box).
# usage: tools/ab_k1.sh WORKLOAD STEPS "ENV1" "ENV2" ...   (ENV like "GF_DOCBLOCK_KB=16024 GF_K1=1")
wl=$1; steps=$2; shift 2
extra=${AB_ARGS:-}
for cfg in "$@"; do
  env $cfg timeout 900 python bench.py --workload $wl $extra --no-cpu-baseline --no-e2e --steps $steps > gpurun_out/ab.log 2>&1
  echo "$wl [$cfg] $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab.log) $(grep -o '"kernel_ms": {[^}]*}' gpurun_out/ab.log) $(grep -o '"frac": [0-9.]*' gpurun_out/ab.log)"
  grep -q ms_per_step gpurun_out/ab.log || tail -5 gpurun_out/ab.log
done
