# Final round-1 refresh of the multi-GPU secondary configs (p2p), 4 GPUs.
O=gpurun_out; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $T --nproc-per-node 2 --master-port 29601 bench_configs.py --config 2 > $O/rf_cfg2h_n2.log 2>&1
timeout 300 $T --nproc-per-node 4 --master-port 29602 bench_configs.py --config 2 > $O/rf_cfg2h_n4.log 2>&1
timeout 400 $T --nproc-per-node 2 --master-port 29603 bench_configs.py --config 5 > $O/rf_cfg5.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29604 bench_configs.py --config 3 > $O/rf_cfg3_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29605 bench_configs.py --config 3 --spmv > $O/rf_cfg3_spmv_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29606 bench_configs.py --config 4 > $O/rf_cfg4_n4.log 2>&1
timeout 400 $T --nproc-per-node 4 --master-port 29607 bench.py --gpus 4 > $O/rf_bench_n4.log 2>&1
