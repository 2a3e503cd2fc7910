O=gpurun_out; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/mq.log 2>&1; echo "rc $?" >> $O/mq.log
