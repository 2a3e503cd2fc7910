# 4-GPU refresh of the final build: full suite, bench N=1/2/4, halo / configs 3-4 at N=4, warp-seq fetch ablation
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2x_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2x_tests_4gpu.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2x_bench_n1.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29631 bench.py --gpus 2 > $O/r2x_bench_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29632 bench.py --gpus 4 > $O/r2x_bench_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29633 bench.py --gpus 4 --dims 2,2,1 --no-e2e > $O/r2x_bench_n4_dims221.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29634 bench.py --gpus 4 --transport nccl --no-e2e > $O/r2x_bench_n4_nccl.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29635 bench_configs.py --config 2 > $O/r2x_cfg2_halo_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29636 bench_configs.py --config 4 > $O/r2x_cfg4_n4.log 2>&1
SFG_CSR_WARP_SEQ=1 timeout 400 $TR --nproc-per-node 4 --master-port 29637 bench_configs.py --config 4 > $O/r2x_cfg4_n4_warpseq.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29638 bench_configs.py --config 3 > $O/r2x_cfg3_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29639 bench_configs.py --config 3 --spmv > $O/r2x_spmv_n4.log 2>&1
