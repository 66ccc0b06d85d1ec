bash tools/ab_k1.sh pubmed 10 "GF_REC_PF=1" "GF_REC_PF=0" "GF_REC_PF=1"
bash tools/ab_k1.sh nytimes 10 "GF_REC_PF=1" "GF_REC_PF=0"
