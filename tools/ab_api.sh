# GPU tests of the phases / one-call API + the API e2e (NYTimes-shape)
o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_phases.py tests/test_gpu_parity.py -q -x -k "phases or export or resident or pinned or sample_chunk" 2>&1 | tail -3
timeout 900 python tools/api_e2e.py --tag ${1:-rX} --out-dir $o > $o/${1:-rX}_api.log 2>&1; echo "api e2e rc=$?"; python -c "
import json; d=json.load(open('$o/${1:-rX}_api_e2e_nytimes.json')); print('api G tok/s', round(d['api_tokens_per_s']/1e9,3), {k: round(v*1e3,2) for k,v in d['mean_seconds'].items()})"
