bash tools/ab_k1.sh pubmed 10 "GF_PREFETCH=1" "GF_PREFETCH=2" "GF_PREFETCH=0" "GF_PREFETCH=1"
bash tools/ab_k1.sh nytimes 10 "GF_PREFETCH=1" "GF_PREFETCH=2"
