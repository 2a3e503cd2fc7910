O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q > $O/quick_ops.log 2>&1
timeout 300 python bench_configs.py --config 1 > $O/quick_cfg1.log 2>&1
timeout 300 python bench_configs.py --config 4 > $O/quick_cfg4.log 2>&1
