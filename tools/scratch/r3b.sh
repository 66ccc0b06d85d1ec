o=gpurun_out
timeout 600 python -m pytest tests/test_gpu_block_phases.py tests/test_gpu_phases.py -q -x 2>&1 | tail -4
for ord in doc word; do
  GF_E2E_ORDER=$ord timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/r3b_$ord.json 2> $o/r3b_$ord.err
  python -c "
import json; d=json.loads([l for l in open('$o/r3b_$ord.json') if l.startswith('{')][-1]); print('$ord', 'value', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), d['e2e']['api'][:60])" || tail -5 $o/r3b_$ord.err
done
GF_E2E_ORDER=doc GF_E2E_PHASES=geo:6 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/r3b_doc6.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('$o/r3b_doc6.json') if l.startswith('{')][-1]); print('doc geo:6', 'e2e', round(d['e2e']['value']/1e9,3))"
