# Ping-pong with 1/2/4 put chunks per CTA (SFG_LL_PUT_LOOP)
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=30120
for l in 1 2 4; do
  p=$((p+1)); SFG_LL_PUT_LOOP=$l timeout 900 $TR --master-port $p bench_configs.py --config 5 > $O/r2fa_loop$l.log 2>&1
done
