O=gpurun_out; mkdir -p $O
for t in p2p nccl; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --transport $t > $O/bench_n2_$t.log 2>&1
done
