# 2 GPUs: halo with the incremental LL receive; compute-sanitizer memcheck over
# the single-GPU op suite (incl. the p2p self-put path) and over the
# process-per-GPU p2p worker (each rank sanitized in its own process).
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29521 bench_configs.py --config 2 --steps 30 > $O/r2m_cfg2_halo_n2.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_ops.py tests/test_gpu_parity2.py -q -x -k "p2p or fig2 or random_all_ops or neighbour or captured or fixtures" > $O/r2m_memcheck_1gpu.log 2>&1; echo "rc=$?" >> $O/r2m_memcheck_1gpu.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29529 --no-python compute-sanitizer --tool memcheck --error-exitcode 99 python tests/mp_worker.py p2p > $O/r2m_memcheck_p2p_2proc.log 2>&1; echo "rc=$?" >> $O/r2m_memcheck_p2p_2proc.log
