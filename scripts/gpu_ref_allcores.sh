O=gpurun_out; mkdir -p $O
nproc > $O/f5_nproc.log; free -g >> $O/f5_nproc.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > $O/f5_bench_ref.log 2>&1; echo "rc $?" >> $O/f5_bench_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29573 bench.py --impl reference --gpus 2 > $O/f5_bench_ref_n2.log 2>&1; echo "rc $?" >> $O/f5_bench_ref_n2.log
