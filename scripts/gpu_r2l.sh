# 4-GPU box: full GPU suite (4-GPU variants), bench at N=1/2/4, halo / configs 3-4 at N=4
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2l_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2l_tests_4gpu.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2l_bench_n1.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29531 bench.py --gpus 2 > $O/r2l_bench_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29532 bench.py --gpus 4 > $O/r2l_bench_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29533 bench.py --gpus 4 --dims 2,2,1 --no-e2e > $O/r2l_bench_n4_dims221.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29534 bench.py --gpus 4 --transport nccl --no-e2e > $O/r2l_bench_n4_nccl.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29535 bench_configs.py --config 2 > $O/r2l_cfg2_halo_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29536 bench_configs.py --config 4 > $O/r2l_cfg4_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29537 bench_configs.py --config 3 > $O/r2l_cfg3_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --impl reference > $O/r2l_bench_ref.log 2>&1
