O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > $O/multi_dsetup.log 2>&1
echo "exit $?" >> $O/multi_dsetup.log
