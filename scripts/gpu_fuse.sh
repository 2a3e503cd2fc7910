O=gpurun_out; mkdir -p $O; : > $O/fuse.log
timeout -s KILL 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ops.py -x -q >> $O/fuse.log 2>&1; echo "rc $?" >> $O/fuse.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for v in fused unfused; do
  if [ $v = unfused ]; then export SFG_P2P_NO_FUSED_UNPACK=1; fi
  timeout 300 $T --master-port 29551 bench_configs.py --config 2 > $O/fuse_cfg2_$v.log 2>&1
  timeout 400 $T --master-port 29552 bench_configs.py --config 5 --max-bytes 2097152 > $O/fuse_cfg5_$v.log 2>&1
done
