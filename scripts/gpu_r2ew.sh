# Same-box A/B: exchange kernel at 2 vs 3 CTAs/SM (halo N=2, 512/1024/2048; ping-pong)
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=30010
for rep in 1 2; do
  for v in c2 c3; do
    cp ab_tmp/_sfgpu_$v.so paper_2102_13018_b200/_sfgpu.so
    for n in 512 1024 2048; do
      p=$((p+1)); timeout 600 $TR --master-port $p bench_configs.py --config 2 --n2 $n --steps 10 > $O/r2ew_${v}_n${n}_r$rep.log 2>&1
    done
  done
done
for v in c2 c3; do
  cp ab_tmp/_sfgpu_$v.so paper_2102_13018_b200/_sfgpu.so
  p=$((p+1)); timeout 900 $TR --master-port $p bench_configs.py --config 5 > $O/r2ew_${v}_cfg5.log 2>&1
done
