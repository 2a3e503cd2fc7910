O=gpurun_out; mkdir -p $O
nproc > $O/tn2.log
SFG_TRACE_SETUP=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-device-setup >> $O/tn2.log 2>&1
