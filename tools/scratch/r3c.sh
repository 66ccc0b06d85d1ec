o=gpurun_out
for ph in geo:9 r0.4:7 r0.35:6 r0.45:8 geo:9; do
  GF_E2E_PHASES=$ph timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/r3c.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('$o/r3c.json') if l.startswith('{')][-1]); print('$ph', 'value', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3))"
done
