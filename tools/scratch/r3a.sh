bash tools/ab_counts.sh r3a "GF_K3_CTAS=0" "GF_K3_CTAS=4" "GF_K3_CTAS=3" "GF_K3_CTAS=0"
