set -u
o=gpurun_out; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/r2b_gputests.log 2>&1; echo "gpu tests: $(tail -3 $o/r2b_gputests.log)"
grep -E "FAILED|passed|failed" $o/r2b_gputests.log | tail -8
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"sample_kernel|phi_rebuild|theta_rebuild|prepare_kernel|context_kernel|ll_reduce|memset" -s 6 -c 36 --csv \
    --log-file $o/r2b_launches_pm.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"sample_kernel|theta_rebuild|phi_rebuild" -s 9 -c 3 \
    -o $o/r2b_pm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $o/r2b_ncu_pm.log 2>&1
echo "pubmed capture rc=$?"
