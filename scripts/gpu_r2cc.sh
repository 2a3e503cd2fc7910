O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_spmv.py -x -q -m gpu > $O/r2cc_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2cc_tests.log
