O=gpurun_out; mkdir -p $O
timeout 300 ./scripts/ll128_bench 500 > $O/r2d_ll128.log 2>&1; echo "rc=$?" >> $O/r2d_ll128.log
CUDA_VISIBLE_DEVICES=0 timeout 300 ./scripts/gather_bench > $O/r2d_gather.log 2>&1; echo "rc=$?" >> $O/r2d_gather.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > $O/r2d_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2d_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29521 bench_configs.py --config 2 > $O/r2d_cfg2_halo_n2.log 2>&1
timeout 600 $TR --master-port 29523 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > $O/r2d_bench_n2.log 2>&1
