O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29521 bench_configs.py --config 2 --steps 30 > $O/r2i_cfg2.log 2>&1
SFG_P2P_NO_FORK=1 timeout 300 $TR --master-port 29522 bench_configs.py --config 2 --steps 30 > $O/r2i_cfg2_nofork.log 2>&1
SFG_P2P_NO_LL128=1 timeout 300 $TR --master-port 29523 bench_configs.py --config 2 --steps 30 > $O/r2i_cfg2_noll.log 2>&1
timeout 300 $TR --master-port 29525 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-device-setup > $O/r2i_bench_n2.log 2>&1
