O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu > $O/r2g_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2g_tests.log
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "threads_of_one or stress or outstanding" > $O/r2g_multi_rep$i.log 2>&1; echo "pytest rc=$?" >> $O/r2g_multi_rep$i.log; done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29521 bench_configs.py --config 2 > $O/r2g_cfg2_halo_n2.log 2>&1
timeout 300 $TR --master-port 29523 bench.py --gpus 2 --steps 20 --warmup 5 > $O/r2g_bench_n2.log 2>&1
