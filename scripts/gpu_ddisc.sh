O=gpurun_out; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dsetup.py -x -q > $O/ddisc_tests.log 2>&1; echo "rc $?" >> $O/ddisc_tests.log
SFG_TRACE_SETUP=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e > $O/ddisc_bench_n4.log 2>&1
