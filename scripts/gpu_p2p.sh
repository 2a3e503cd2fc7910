O=gpurun_out; mkdir -p $O
set -x
timeout 300 python -m pytest tests/test_gpu_ops.py -x -q > $O/p2p_single.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/p2p_multi.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > $O/bench_n1.log 2>&1
for t in p2p nccl; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench_configs.py --config 2 --transport $t > $O/cfg2h_$t.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench_configs.py --config 5 --transport $t > $O/cfg5_$t.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 2 --transport $t > $O/bench_n2_$t.log 2>&1
done
