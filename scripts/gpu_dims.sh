O=gpurun_out; mkdir -p $O
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 4 --dims 2,2,1 > $O/d221.log 2>&1
SFG_NO_COUPLED_SPLIT=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 4 --dims 2,2,1 > $O/d221_nosplit.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29593 bench.py --gpus 4 --dims 4,1,1 > $O/d411.log 2>&1
