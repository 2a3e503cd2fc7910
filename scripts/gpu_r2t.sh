O=gpurun_out; mkdir -p $O
timeout 120 python scripts/halo_threads.py > $O/r2t_halo_threads.log 2>&1
SFG_P2P_NO_FORK=1 timeout 120 python scripts/halo_threads.py > $O/r2t_halo_threads_nofork.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29561 bench_configs.py --config 2 --steps 30 > $O/r2t_cfg2.log 2>&1
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "threads_of_one or stress or outstanding or teardown or g2l" > $O/r2t_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2t_tests.log
