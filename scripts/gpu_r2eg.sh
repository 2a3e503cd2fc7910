O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_multi.py -x -q -m gpu -k "spmv" > $O/r2eg_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2eg_tests.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_configs.py --config 3 --spmv > $O/r2eg_spmv_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29651 bench_configs.py --config 3 --spmv > $O/r2eg_spmv_n2.log 2>&1
