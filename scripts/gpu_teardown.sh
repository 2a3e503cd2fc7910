O=gpurun_out; mkdir -p $O; : > $O/teardown.log
echo "== without quiesce" >> $O/teardown.log
SFG_P2P_NO_QUIESCE=1 timeout -s KILL 120 python -m pytest tests/test_gpu_multi.py -x -q -k teardown >> $O/teardown.log 2>&1; echo "rc $?" >> $O/teardown.log
echo "== with quiesce" >> $O/teardown.log
timeout -s KILL 120 python -m pytest tests/test_gpu_multi.py -x -q -k teardown >> $O/teardown.log 2>&1; echo "rc $?" >> $O/teardown.log
echo "== full multi" >> $O/teardown.log
timeout -s KILL 400 python -m pytest tests/test_gpu_multi.py -x -q >> $O/teardown.log 2>&1; echo "rc $?" >> $O/teardown.log
