o=gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel" -s 6 -c 1 \
  -o $o/r3e_shard_k1 python bench.py --shard 0/8 --steps 2 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "rc=$?"
