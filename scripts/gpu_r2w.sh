O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "protocol_per_unit or threads_of_one" > $O/r2w_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2w_tests.log
