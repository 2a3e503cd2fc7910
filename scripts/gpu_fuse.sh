O=gpurun_out; mkdir -p $O; : > $O/fuse.log
timeout -s KILL 400 python -m pytest tests/test_gpu_multi.py -x -q >> $O/fuse.log 2>&1; echo "rc $?" >> $O/fuse.log
for v in fused unfused; do
  if [ $v = unfused ]; then export SFG_P2P_NO_FUSED_UNPACK=1; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench_configs.py --config 2 > $O/fuse_cfg2_$v.log 2>&1
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 > $O/fuse_bench_$v.log 2>&1
done
