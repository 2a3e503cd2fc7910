O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
SFG_TRACE_LAUNCHES=100000 timeout 300 $TR --master-port 29571 bench_configs.py --config 2 --steps 10 > $O/r2u_cfg2_trace.log 2>&1
SFG_TRACE_LAUNCHES=100000 SFG_P2P_NO_FORK=1 timeout 300 $TR --master-port 29572 bench_configs.py --config 2 --steps 10 > $O/r2u_cfg2_trace_nofork.log 2>&1
