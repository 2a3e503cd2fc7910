O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_ops.py -x -q > $O/spmv_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/spmv_multi.log 2>&1
timeout 600 python bench_configs.py --config 3 --spmv > $O/cfg3_spmv_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench_configs.py --config 3 --spmv > $O/cfg3_spmv_n2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench_configs.py --config 2 > $O/cfg2h_p2p.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 bench_configs.py --config 5 > $O/cfg5_p2p.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29564 bench.py --gpus 2 > $O/bench_n2_p2p.log 2>&1
