# LL128 put chunks per CTA sweep (SFG_LL_PUT_LOOP) on the halo at N=2: 512^3 / 1024^3 / 2048^3
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=29940
for l in 1 2 4 8; do
  for n in 512 1024 2048; do
    p=$((p+1)); SFG_LL_PUT_LOOP=$l timeout 600 $TR --master-port $p bench_configs.py --config 2 --n2 $n --steps 10 > $O/r2et_loop${l}_n$n.log 2>&1
  done
done
