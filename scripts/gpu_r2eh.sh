# LL128 receive poll back-off sweep: halo-only config 2 at N=2 (512^3: 2 MB, 1024^3: 8 MB per direction)
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=29700
for ns in 20 0 80 200 500 1000; do
  for n in 512 1024; do
    p=$((p+1))
    SFG_LL_POLL_NS=$ns timeout 300 $TR --master-port $p bench_configs.py --config 2 --n2 $n > $O/r2eh_poll${ns}_n$n.log 2>&1
  done
done
