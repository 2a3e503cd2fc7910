# PDL for End folds right behind the exchange launch: halo N=2/N=4, bench N=2/N=4, config 4 N=4, multi-GPU tests
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity2.py -x -q -m gpu > $O/r2ez_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2ez_tests.log
timeout 300 $TR --nproc-per-node 4 --master-port 30101 bench_configs.py --config 2 > $O/r2ez_cfg2_n4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 30102 bench_configs.py --config 2 > $O/r2ez_cfg2_n2.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 30103 bench.py --gpus 2 --no-e2e > $O/r2ez_bench_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 30104 bench.py --gpus 4 --no-e2e > $O/r2ez_bench_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 30105 bench_configs.py --config 4 > $O/r2ez_cfg4_n4.log 2>&1
