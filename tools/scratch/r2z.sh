ALT=$PWD/paper_1803_04631_b200/_lib/alt/libgfb200.so
bash tools/ab_k1.sh pubmed 10 "GF_X=new" "GF_LIB=$ALT" "GF_X=new" "GF_LIB=$ALT"
bash tools/ab_k1.sh nytimes 10 "GF_X=new" "GF_LIB=$ALT"
AB_ARGS="--shard 0/8" bash tools/ab_k1.sh pubmed 10 "GF_X=new" "GF_LIB=$ALT"
