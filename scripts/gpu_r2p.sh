O=gpurun_out; mkdir -p $O
timeout 120 python scripts/halo_threads.py > $O/r2p_halo_threads.log 2>&1
SFG_P2P_NO_FORK=1 timeout 120 python scripts/halo_threads.py > $O/r2p_halo_threads_nofork.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 120 ./scripts/tma_gather_bench > $O/r2p_tma_gather.log 2>&1; echo "rc=$?" >> $O/r2p_tma_gather.log
