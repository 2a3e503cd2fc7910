# LL128 p2p path: multi-GPU parity, halo exchange, ping-pong; configs 1/4 graph timing + CPU baselines
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ops.py -x -q -m gpu > $O/r2c_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2c_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29521 bench_configs.py --config 2 > $O/r2c_cfg2_halo_n2.log 2>&1
timeout 900 $TR --master-port 29522 bench_configs.py --config 5 --cpu > $O/r2c_cfg5_n2.log 2>&1
timeout 600 $TR --master-port 29523 bench.py --gpus 2 --steps 20 --warmup 5 > $O/r2c_bench_n2.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 1 --cpu > $O/r2c_cfg1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 4 --cpu > $O/r2c_cfg4.log 2>&1
