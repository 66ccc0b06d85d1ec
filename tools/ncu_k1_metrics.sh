#!/bin/bash
# targeted ncu metrics of one K1 launch (GPU box).  usage: tools/ncu_k1_metrics.sh WORKLOAD TAG "ENV"
wl=$1; tag=$2; cfg=$3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active
env $cfg timeout 1200 ncu --metrics $M --clock-control none -k regex:"sample_kernel|theta_rebuild" -s 8 -c 2 --csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$tag.csv 2> gpurun_out/ncu_$tag.err
python - gpurun_out/ncu_$tag.csv "$tag" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
for r in rows[1:]:
    print(sys.argv[2], r[ki][:28], r[mi], r[vi])
PY
