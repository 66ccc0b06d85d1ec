# e2e regression check + K2/K3 source-level capture (round 2, session 3)
o=gpurun_out; mkdir -p $o
timeout 120 python tools/scratch/pcie.py > $o/r2l_pcie.log 2>&1; cat $o/r2l_pcie.log
for ph in geo:9 1; do
  GF_E2E_PHASES=$ph timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/r2l_e2e_$ph.json 2>/dev/null
  python -c "
import json,sys; d=json.loads([l for l in open('$o/r2l_e2e_$ph.json') if l.startswith('{')][-1]); print('$ph', 'value', d['value']/1e9, 'e2e', d['e2e']['value']/1e9)"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"theta_rebuild|phi_rebuild" -s 4 -c 2 \
  -o $o/r2l_k23 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "ncu rc=$?"
python profiles/ncu_summary.py $o/r2l_k23.ncu-rep 40 > $o/r2l_k23.txt 2>&1; head -5 $o/r2l_k23.txt
timeout 900 python tools/api_e2e.py --tag r2l --out-dir $o > $o/r2l_api.log 2>&1; echo "api e2e rc=$?"; tail -c 1500 $o/r2l_api.log
