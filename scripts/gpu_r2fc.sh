O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "torchrun or wide" > $O/r2fc_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2fc_tests.log
