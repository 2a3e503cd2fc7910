O=gpurun_out; mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
timeout 300 python bench_configs.py --config 1 > $O/r2bb_cfg1.log 2>&1
timeout 400 python bench_configs.py --config 4 > $O/r2bb_cfg4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_parity2.py -x -q -m gpu > $O/r2bb_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2bb_tests.log
