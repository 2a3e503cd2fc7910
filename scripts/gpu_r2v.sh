O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ops.py -x -q -m gpu > $O/r2v_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2v_tests.log
timeout 300 $TR --master-port 29581 bench_configs.py --config 2 --steps 30 > $O/r2v_cfg2.log 2>&1
timeout 900 $TR --master-port 29582 bench_configs.py --config 5 --cpu > $O/r2v_cfg5.log 2>&1
