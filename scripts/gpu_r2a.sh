# Round 2, first 2-GPU call: whole GPU suite (new parity2 + multi-GPU full
# size), LL128 microbenchmark, bench N=1 and N=2.
O=gpurun_out; mkdir -p $O
nvidia-smi topo -m > $O/topo.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/r2a_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2a_gpu_tests.log
timeout 300 ./scripts/ll128_bench 2000 > $O/r2a_ll128.log 2>&1; echo "rc=$?" >> $O/r2a_ll128.log
timeout 400 python bench.py --steps 20 --warmup 5 > $O/r2a_bench_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > $O/r2a_bench_n2.log 2>&1
