set -u
o=gpurun_out; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/r2c_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $o/r2c_smoke.log)"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/r2c_gputests.log 2>&1; echo "gpu tests: $(tail -1 $o/r2c_gputests.log)"
grep -E "^FAILED|^ERROR" $o/r2c_gputests.log | head -20
