o=gpurun_out; mkdir -p $o
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"theta_rebuild|phi_rebuild" -s 4 -c 2 \
  -o $o/r2o_k23 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "ncu rc=$?"
python profiles/ncu_summary.py $o/r2o_k23.ncu-rep 30 > $o/r2o_k23.txt 2>&1; head -30 $o/r2o_k23.txt
