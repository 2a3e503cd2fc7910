O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "random_delays" > $O/r2dd_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2dd_tests.log
