O=gpurun_out; mkdir -p $O
for ns in 20 100 400 1000; do SFG_LL_POLL_NS=$ns SFG_P2P_NO_FORK=1 timeout 120 python scripts/halo_threads.py > $O/r2q_halo_poll$ns.log 2>&1; done
SFG_P2P_NO_LL128=1 SFG_P2P_NO_FORK=1 timeout 120 python scripts/halo_threads.py > $O/r2q_halo_flag.log 2>&1
