o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/r2m_gputests.log 2>&1; echo "gpu tests: $(tail -1 $o/r2m_gputests.log)"; grep -E "^FAILED|^ERROR|Error" $o/r2m_gputests.log | head -5
for wl in pubmed nytimes; do
timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > $o/r2m_bench_$wl.json 2> $o/r2m_bench_$wl.err
python - $wl <<'PY'
import json, sys
d=json.loads([l for l in open(f'gpurun_out/r2m_bench_{sys.argv[1]}.json') if l.startswith('{')][-1])
k=d['kernels']; print(sys.argv[1], 'value', round(d['value']/1e9,3), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e9,3), 'K1', round(d['kernel_ms']['sample'],2), 'K2', round(k['phi_rebuild']['ms'],3), 'K3', round(k['theta_rebuild']['ms'],3), 'in_step', k['in_step_ms'])
PY
done
