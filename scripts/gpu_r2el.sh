# Message-order test + config 4 at N=2/4 and config 3 at N=4 on the committed build
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_parity2.py tests/test_gpu_dsetup.py -x -q -m gpu > $O/r2el_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2el_tests.log
timeout 400 $TR --nproc-per-node 4 --master-port 29851 bench_configs.py --config 4 > $O/r2el_cfg4_n4.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29852 bench_configs.py --config 4 > $O/r2el_cfg4_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29853 bench_configs.py --config 3 > $O/r2el_cfg3_n4.log 2>&1
