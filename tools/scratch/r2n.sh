o=gpurun_out; mkdir -p $o
timeout 300 compute-sanitizer --tool memcheck --show-backtrace no python tools/scratch/repro_iam.py > $o/r2n_memcheck.log 2>&1; echo rc=$?; head -30 $o/r2n_memcheck.log
