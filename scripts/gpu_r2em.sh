# Warp limit at exactly 32768 roots per rank (config 4 at N=2)
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SFG_CSR_WARP_LIMIT=32769 timeout 400 $TR --nproc-per-node 2 --master-port 29861 bench_configs.py --config 4 > $O/r2em_cfg4_n2_wl32769.log 2>&1
