O=gpurun_out; mkdir -p $O
timeout 400 python bench.py > $O/bds_n1.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > $O/bds_n2.log 2>&1
