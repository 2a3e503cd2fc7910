# One-shot forms (no stream fork): full GPU suite, halo config 2 / ping-pong config 5 at N=2, bench N=2/4
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -x -q -m gpu > $O/r2ep_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2ep_tests_4gpu.log
timeout 300 $TR --nproc-per-node 2 --master-port 29901 bench_configs.py --config 2 > $O/r2ep_cfg2_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29902 bench_configs.py --config 2 > $O/r2ep_cfg2_n4.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29903 bench_configs.py --config 5 > $O/r2ep_cfg5_n2.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29904 bench.py --gpus 2 > $O/r2ep_bench_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29905 bench.py --gpus 4 > $O/r2ep_bench_n4.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29906 bench_configs.py --config 2 --n2 2048 --steps 10 > $O/r2ep_cfg2_2048_n2.log 2>&1
