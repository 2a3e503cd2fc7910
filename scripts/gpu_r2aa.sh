O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "not torchrun and not 512" > $O/r2aa_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2aa_tests.log
timeout 300 $TR --master-port 29601 bench_configs.py --config 2 --steps 30 > $O/r2aa_cfg2_512.log 2>&1
timeout 600 $TR --master-port 29602 bench_configs.py --config 2 --n2 1024 --steps 20 > $O/r2aa_cfg2_1024.log 2>&1
timeout 900 $TR --master-port 29603 bench_configs.py --config 2 --n2 2048 --steps 10 > $O/r2aa_cfg2_2048.log 2>&1
