O=gpurun_out; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/f6_bench_n1.log 2>&1; echo "rc $?" >> $O/f6_bench_n1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29575 bench.py --gpus 2 > $O/f6_bench_n2.log 2>&1; echo "rc $?" >> $O/f6_bench_n2.log
