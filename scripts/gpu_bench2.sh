O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q > $O/ops_q.log 2>&1
for t in p2p nccl; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --transport $t > $O/bench_n2_$t.log 2>&1
done
SFG_NO_COUPLED_SPLIT=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 > $O/bench_n2_nosplit.log 2>&1
