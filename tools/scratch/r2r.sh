o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/r2r_gputests.log 2>&1; echo "gpu tests: $(tail -1 $o/r2r_gputests.log)"; grep -E "^FAILED|^ERROR" $o/r2r_gputests.log | head -5
bash tools/ab_k1.sh pubmed 10 "GF_CTX_TMA=1" "GF_CTX_TMA=0" "GF_CTX_TMA=1"
AB_ARGS="--shard 0/8" bash tools/ab_k1.sh pubmed 10 "GF_CTX_TMA=1" "GF_CTX_TMA=0"
