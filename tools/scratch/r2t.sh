o=gpurun_out
for ph in geo:9 geo:6 geo:12 8; do
  GF_E2E_PHASES=$ph timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/r2t_$ph.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('$o/r2t_$ph.json') if l.startswith('{')][-1]); print('$ph', 'value', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3))"
done
timeout 600 python tools/scratch/e2e_probe.py > $o/r2t_probe.log 2>&1; cat $o/r2t_probe.log | tail -20
