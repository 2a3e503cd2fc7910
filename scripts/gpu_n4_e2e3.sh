O=gpurun_out; mkdir -p $O
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29577 bench.py --gpus 4 > $O/f7_bench_n4.log 2>&1; echo "rc $?" >> $O/f7_bench_n4.log
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29578 bench.py --impl reference --gpus 4 > $O/f7_bench_ref_n4.log 2>&1; echo "rc $?" >> $O/f7_bench_ref_n4.log
