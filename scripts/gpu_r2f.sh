O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29521 bench_configs.py --config 2 > $O/r2f_cfg2_halo_n2.log 2>&1
SFG_P2P_NO_LL128=1 timeout 300 $TR --master-port 29522 bench_configs.py --config 2 > $O/r2f_cfg2_halo_n2_noll.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > $O/r2f_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2f_tests.log
timeout 300 $TR --master-port 29523 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > $O/r2f_bench_n2.log 2>&1
