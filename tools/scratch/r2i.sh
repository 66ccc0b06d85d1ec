o=gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dist-backend gloo --workload nytimes --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $o/r2i_n2_gloo.json 2> $o/r2i_n2_gloo.err; echo "n2 gloo rc=$?"; tail -c 400 $o/r2i_n2_gloo.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $o/r2i_n2_ref.json 2> $o/r2i_n2_ref.err; echo "n2 ref rc=$?"; tail -c 300 $o/r2i_n2_ref.json
GF_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --workload nytimes --steps 3 --warmup 3 --no-cpu-baseline > $o/r2i_n1_nccl.json 2> $o/r2i_n1_nccl.err; echo "n1 nccl rc=$?"; tail -c 300 $o/r2i_n1_nccl.json
bash tools/ab_counts.sh r2i "GF_K3_MINB=5"
