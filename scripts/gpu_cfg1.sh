O=gpurun_out; mkdir -p $O
timeout 400 python bench_configs.py --config 1 > $O/cfg1_na.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py -x -q > $O/cfg1_na_tests.log 2>&1; echo "rc $?" >> $O/cfg1_na_tests.log
