O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "protocol or g2l_halo or spmv" > $O/r2eq_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2eq_tests.log
