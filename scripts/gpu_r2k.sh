O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
SFG_TRACE_LAUNCHES=100000 timeout 300 $TR --master-port 29521 bench_configs.py --config 2 --steps 10 > $O/r2k_cfg2_trace.log 2>&1
timeout 300 $TR --master-port 29522 bench_configs.py --config 2 --steps 30 > $O/r2k_cfg2.log 2>&1
SFG_P2P_NO_FORK=1 timeout 300 $TR --master-port 29523 bench_configs.py --config 2 --steps 30 > $O/r2k_cfg2_nofork.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "threads_of_one or stress or outstanding or g2l or teardown" > $O/r2k_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2k_tests.log
