# LL128 interleave rule A/B: config 4 at N=4 (indexed puts) and the halo (structured puts)
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > $O/r2ei_tests_multi.log 2>&1; echo "pytest rc=$?" >> $O/r2ei_tests_multi.log
timeout 400 $TR --nproc-per-node 4 --master-port 29821 bench_configs.py --config 4 > $O/r2ei_cfg4_n4.log 2>&1
SFG_LL_INTERLEAVE=all timeout 400 $TR --nproc-per-node 4 --master-port 29822 bench_configs.py --config 4 > $O/r2ei_cfg4_n4_ilvall.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29823 bench_configs.py --config 2 > $O/r2ei_cfg2_512_n2.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29824 bench_configs.py --config 2 --n2 2048 --steps 10 > $O/r2ei_cfg2_2048_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29825 bench_configs.py --config 2 > $O/r2ei_cfg2_512_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29826 bench_configs.py --config 3 > $O/r2ei_cfg3_n4.log 2>&1
