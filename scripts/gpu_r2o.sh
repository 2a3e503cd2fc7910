O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for i in 1 2; do
timeout 300 $TR --master-port 2952$i bench_configs.py --config 2 --steps 30 > $O/r2o_cfg2_$i.log 2>&1
SFG_P2P_NO_FORK=1 timeout 300 $TR --master-port 2953$i bench_configs.py --config 2 --steps 30 > $O/r2o_cfg2_nofork_$i.log 2>&1
done
SFG_TRACE_LAUNCHES=100000 timeout 300 $TR --master-port 29541 bench_configs.py --config 2 --steps 10 > $O/r2o_cfg2_trace.log 2>&1
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "threads_of_one or stress or outstanding or teardown" > $O/r2o_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2o_tests.log
