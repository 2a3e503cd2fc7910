O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dsetup.py -x -q -s > $O/dsetup_tests.log 2>&1
echo "exit $?" >> $O/dsetup_tests.log
SFG_TRACE_SETUP=1 timeout 300 python scripts/trace_setup.py 512 both > $O/dsetup_trace.log 2>&1
