O=gpurun_out; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 4 --master-port 29611 bench_configs.py --config 4 > $O/wl_cfg4_n4.log 2>&1
timeout 400 python bench_configs.py --config 4 > $O/wl_cfg4_n1.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ops.py tests/test_gpu_fullsize.py -x -q > $O/wl_tests.log 2>&1; echo "rc $?" >> $O/wl_tests.log
