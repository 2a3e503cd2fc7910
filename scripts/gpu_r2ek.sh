# Warp-per-root End folds (roots with remote contributions) and the warp limit: config 4 at N=1/2/4
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity2.py tests/test_gpu_ops.py -x -q -m gpu > $O/r2ek_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2ek_tests.log
timeout 400 $TR --nproc-per-node 4 --master-port 29841 bench_configs.py --config 4 > $O/r2ek_cfg4_n4.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29842 bench_configs.py --config 4 > $O/r2ek_cfg4_n2.log 2>&1
SFG_CSR_WARP_LIMIT=65537 timeout 400 $TR --nproc-per-node 2 --master-port 29843 bench_configs.py --config 4 > $O/r2ek_cfg4_n2_wl64k.log 2>&1
SFG_CSR_WARP_LIMIT=65537 CUDA_VISIBLE_DEVICES=0 timeout 400 python bench_configs.py --config 4 > $O/r2ek_cfg4_n1_wl64k.log 2>&1
