bash tools/ab_k1.sh pubmed 10 "GF_K1=0" "GF_K1=4" "GF_K1=5" "GF_K1=0"
bash tools/ab_k1.sh nytimes 10 "GF_K1=0" "GF_K1=4" "GF_K1=5"
AB_ARGS="--shard 0/8" bash tools/ab_k1.sh pubmed 10 "GF_K1=0" "GF_K1=4"
