O=gpurun_out; mkdir -p $O
for t in p2p nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench_configs.py --config 3 --transport $t > $O/cfg3_n4_$t.log 2>&1
done
