# Final 4-GPU refresh of the round-2 build: full GPU suite, smoke, bench N=1/2/4 (+ reference
# arm, dims 2,2,1, nccl), configs 1-5, SpMV N=1/2/4, ncu launch list of the headline bench.
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r2f_box.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/r2f_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2f_tests_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2f_smoke.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2f_bench_n1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > $O/r2f_bench_ref.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29801 bench.py --gpus 2 > $O/r2f_bench_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 > $O/r2f_bench_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --dims 2,2,1 --no-e2e > $O/r2f_bench_n4_dims221.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --transport nccl --no-e2e > $O/r2f_bench_n4_nccl.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench_configs.py --config 1 > $O/r2f_cfg1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench_configs.py --config 4 > $O/r2f_cfg4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29805 bench_configs.py --config 2 > $O/r2f_cfg2_halo_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29806 bench_configs.py --config 2 > $O/r2f_cfg2_halo_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29807 bench_configs.py --config 4 > $O/r2f_cfg4_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29808 bench_configs.py --config 3 > $O/r2f_cfg3_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_configs.py --config 3 --spmv > $O/r2f_spmv_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29809 bench_configs.py --config 3 --spmv > $O/r2f_spmv_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29810 bench_configs.py --config 3 --spmv > $O/r2f_spmv_n4.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29811 bench_configs.py --config 5 > $O/r2f_cfg5_n2.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2f_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2f_ncu_launches.log 2>&1
