# Final build: full GPU suite (4 GPUs), smoke, bench N=1/4 (+dims 2,2,1, nccl), halo N=4, SpMV N=1/2/4, ncu launch list
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2h_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2h_tests_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2h_smoke.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2h_bench_n1.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29931 bench.py --gpus 4 > $O/r2h_bench_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29932 bench.py --gpus 4 --dims 2,2,1 --no-e2e > $O/r2h_bench_n4_dims221.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29933 bench.py --gpus 4 --transport nccl --no-e2e > $O/r2h_bench_n4_nccl.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29934 bench_configs.py --config 2 > $O/r2h_cfg2_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_configs.py --config 3 --spmv > $O/r2h_spmv_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29935 bench_configs.py --config 3 --spmv > $O/r2h_spmv_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29936 bench_configs.py --config 3 --spmv > $O/r2h_spmv_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2h_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2h_ncu_launches.log 2>&1
