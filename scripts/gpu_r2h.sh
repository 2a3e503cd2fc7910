O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29521 bench_configs.py --config 2 --steps 30 > $O/r2h_cfg2.log 2>&1
SFG_P2P_NO_FORK=1 timeout 300 $TR --master-port 29522 bench_configs.py --config 2 --steps 30 > $O/r2h_cfg2_nofork.log 2>&1
SFG_P2P_NO_LL128=1 timeout 300 $TR --master-port 29523 bench_configs.py --config 2 --steps 30 > $O/r2h_cfg2_noll.log 2>&1
SFG_P2P_NO_LL128=1 SFG_P2P_NO_FORK=1 timeout 300 $TR --master-port 29524 bench_configs.py --config 2 --steps 30 > $O/r2h_cfg2_noll_nofork.log 2>&1
timeout 120 ./scripts/ll128_bench 10 > $O/r2h_ll128.log 2>&1
