O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity2.py tests/test_gpu_ops.py -x -q -m gpu > $O/r2fd_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2fd_tests.log
