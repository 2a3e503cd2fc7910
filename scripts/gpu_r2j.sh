O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
SFG_TRACE_LAUNCHES=100000 timeout 300 $TR --master-port 29521 bench_configs.py --config 2 --steps 10 > $O/r2j_cfg2_trace.log 2>&1
