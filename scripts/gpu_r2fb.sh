# Config 3 ghost SF at N=4 with the one-shot forms beside split-phase
O=gpurun_out; mkdir -p $O
timeout 400 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 30131 bench_configs.py --config 3 > $O/r2fb_cfg3_n4.log 2>&1
