o=gpurun_out
for ph in geo:9 r0.45:8 geo:9 r0.45:8 r0.5:10; do
  GF_E2E_PHASES=$ph timeout 600 python bench.py --workload nytimes --steps 10 --warmup 3 --no-cpu-baseline > $o/r3f.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('$o/r3f.json') if l.startswith('{')][-1]); print('nyt $ph', 'value', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3))"
done
