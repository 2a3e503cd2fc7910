O=gpurun_out; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_dsetup.py -x -q > $O/dsetup_tests.log 2>&1
echo "exit $?" >> $O/dsetup_tests.log
