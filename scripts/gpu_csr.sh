O=gpurun_out; mkdir -p $O
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > $O/csr_gpu_tests.log 2>&1
echo "exit $?" >> $O/csr_gpu_tests.log
SFG_TRACE_SETUP=1 timeout 400 python bench_configs.py --config 4 > $O/csr_cfg4.log 2>&1
SFG_TRACE_SETUP=1 timeout 400 python bench_configs.py --config 1 > $O/csr_cfg1.log 2>&1
