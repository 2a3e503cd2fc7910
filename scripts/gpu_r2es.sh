# PDL on exchange launches only: bench N=2 (twice), halo N=2, config 5, GPU multi tests
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > $O/r2es_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2es_tests.log
timeout 400 $TR --master-port 29921 bench.py --gpus 2 > $O/r2es_bench_n2.log 2>&1
SFG_NO_PDL=1 timeout 400 $TR --master-port 29922 bench.py --gpus 2 > $O/r2es_bench_n2_nopdl.log 2>&1
timeout 300 $TR --master-port 29923 bench_configs.py --config 2 > $O/r2es_cfg2_n2.log 2>&1
timeout 900 $TR --master-port 29924 bench_configs.py --config 5 > $O/r2es_cfg5_n2.log 2>&1
