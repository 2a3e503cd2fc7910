# Same-box A/B: committed build vs the put-loop build (loop 1 and 2), halo N=2 512^3 / 2048^3, alternating
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=29960
for rep in 1 2; do
  for v in old new new2; do
    case $v in old) cp ab_tmp/_sfgpu_old.so paper_2102_13018_b200/_sfgpu.so; env="";; new) cp ab_tmp/_sfgpu_new.so paper_2102_13018_b200/_sfgpu.so; env="";; new2) cp ab_tmp/_sfgpu_new.so paper_2102_13018_b200/_sfgpu.so; env="SFG_LL_PUT_LOOP=2";; esac
    for n in 512 2048; do
      p=$((p+1)); env $env timeout 600 $TR --master-port $p bench_configs.py --config 2 --n2 $n --steps 10 > $O/r2eu_${v}_n${n}_r$rep.log 2>&1
    done
  done
done
