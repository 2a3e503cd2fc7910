# Message order (remote groups sorted by root offset): full GPU suite, config 4 / 3 at N=4 with and without, halo, bench N=4
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -x -q -m gpu > $O/r2ej_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2ej_tests_4gpu.log
timeout 400 $TR --nproc-per-node 4 --master-port 29831 bench_configs.py --config 4 > $O/r2ej_cfg4_n4.log 2>&1
SFG_NO_WIRE_SORT=1 timeout 400 $TR --nproc-per-node 4 --master-port 29832 bench_configs.py --config 4 > $O/r2ej_cfg4_n4_nowire.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29833 bench_configs.py --config 4 > $O/r2ej_cfg4_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29834 bench_configs.py --config 3 > $O/r2ej_cfg3_n4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29835 bench_configs.py --config 2 > $O/r2ej_cfg2_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29836 bench.py --gpus 4 --no-e2e > $O/r2ej_bench_n4.log 2>&1
