# Same-box A/B: wide exchange kernel at 3 vs 4 CTAs/SM (halo N=2 1024^3 / 2048^3)
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=30080
for rep in 1 2; do
  for v in c3 c4; do
    cp ab_tmp/_sfgpu_$v.so paper_2102_13018_b200/_sfgpu.so
    for n in 1024 2048; do
      p=$((p+1)); timeout 600 $TR --master-port $p bench_configs.py --config 2 --n2 $n --steps 10 > $O/r2ey_${v}_n${n}_r$rep.log 2>&1
    done
  done
done
