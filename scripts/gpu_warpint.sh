O=gpurun_out; mkdir -p $O
timeout 400 python bench_configs.py --config 4 > $O/wi_cfg4_base.log 2>&1
SFG_CSR_WARP_INT=1 timeout 400 python bench_configs.py --config 4 > $O/wi_cfg4_warp.log 2>&1
SFG_CSR_WARP_INT=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_ops.py -x -q > $O/wi_tests.log 2>&1
