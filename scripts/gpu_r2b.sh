O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2b_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2b_gpu_tests.log
timeout 300 ./scripts/gather_bench > $O/r2b_gather.log 2>&1; echo "rc=$?" >> $O/r2b_gather.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/r2b_bench_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > $O/r2b_bench_n2.log 2>&1
