bash tools/ab_counts.sh r2h "GF_K3_SHORTSORT=0" "GF_K3_SHORTSORT=1"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"theta_rebuild" -s 4 -c 1 -o gpurun_out/r2h_k3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
