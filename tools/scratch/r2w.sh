o=gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel" -s 6 -c 1 \
  -o $o/r2w_k1 python bench.py --steps 2 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "rc=$?"
python profiles/ncu_summary.py $o/r2w_k1.ncu-rep 12 > $o/r2w_k1.txt 2>&1; head -40 $o/r2w_k1.txt
