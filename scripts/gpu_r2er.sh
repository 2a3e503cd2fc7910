# Programmatic dependent launch: full GPU suite, halo N=2/N=4, configs 1/4 N=1, bench N=1/2, PDL ablation
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -x -q -m gpu > $O/r2er_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2er_tests_4gpu.log
timeout 300 $TR --nproc-per-node 2 --master-port 29911 bench_configs.py --config 2 > $O/r2er_cfg2_n2.log 2>&1
SFG_NO_PDL=1 timeout 300 $TR --nproc-per-node 2 --master-port 29912 bench_configs.py --config 2 > $O/r2er_cfg2_n2_nopdl.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29913 bench_configs.py --config 2 > $O/r2er_cfg2_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench_configs.py --config 1 > $O/r2er_cfg1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench_configs.py --config 4 > $O/r2er_cfg4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2er_bench_n1.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29914 bench.py --gpus 2 > $O/r2er_bench_n2.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29915 bench_configs.py --config 5 > $O/r2er_cfg5_n2.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29916 bench_configs.py --config 3 --spmv > $O/r2er_spmv_n2.log 2>&1
