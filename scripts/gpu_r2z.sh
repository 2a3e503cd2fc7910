O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29591 bench_configs.py --config 2 --n2 1024 --steps 20 > $O/r2z_cfg2_halo_1024_n2.log 2>&1
timeout 900 $TR --master-port 29592 bench_configs.py --config 2 --n2 2048 --steps 10 > $O/r2z_cfg2_halo_2048_n2.log 2>&1
