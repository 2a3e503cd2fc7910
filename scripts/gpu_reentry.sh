O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/f4_smoke.log 2>&1; echo "rc $?" >> $O/f4_smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/f4_gpu_tests.log 2>&1; echo "rc $?" >> $O/f4_gpu_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/f4_bench_n1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --impl reference > $O/f4_bench_ref.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 > $O/f4_bench_n2.log 2>&1
