# 3 CTAs/SM exchange kernel for launches >= 65536 LL lines: same-box A/B vs the committed 2-CTA build; put-loop under it
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=30040
for v in c2 new new_loop1; do
  case $v in c2) cp ab_tmp/_sfgpu_c2.so paper_2102_13018_b200/_sfgpu.so; env="";; new) cp ab_tmp/_sfgpu_new.so paper_2102_13018_b200/_sfgpu.so; env="";; new_loop1) cp ab_tmp/_sfgpu_new.so paper_2102_13018_b200/_sfgpu.so; env="SFG_LL_PUT_LOOP=1";; esac
  for n in 512 1024 2048; do
    p=$((p+1)); env $env timeout 600 $TR --master-port $p bench_configs.py --config 2 --n2 $n --steps 10 > $O/r2ex_${v}_n${n}.log 2>&1
  done
done
cp ab_tmp/_sfgpu_new.so paper_2102_13018_b200/_sfgpu.so
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > $O/r2ex_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2ex_tests.log
p=$((p+1)); timeout 900 $TR --master-port $p bench_configs.py --config 5 > $O/r2ex_cfg5.log 2>&1
