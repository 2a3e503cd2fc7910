O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/multi_n4.log 2>&1
for t in p2p nccl; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --transport $t > $O/bench_n4_$t.log 2>&1
done
