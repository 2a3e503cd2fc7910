O=gpurun_out; mkdir -p $O
timeout 200 ./scripts/ll128_bench 300 > $O/r2e_ll128.log 2>&1; echo "rc=$?" >> $O/r2e_ll128.log
timeout 900 python -m pytest tests -x -q -m gpu > $O/r2e_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2e_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29521 bench_configs.py --config 2 > $O/r2e_cfg2_halo_n2.log 2>&1
timeout 300 $TR --master-port 29523 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > $O/r2e_bench_n2.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_configs.py --config 1 > $O/r2e_cfg1.log 2>&1
CUDA_VISIBLE_DEVICES=0 SFG_NO_SOLO=1 timeout 300 python bench_configs.py --config 1 > $O/r2e_cfg1_nosolo.log 2>&1
