# Same-box A/B: committed build vs put-loop-for-op-receives build; multi-GPU tests on the new build
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=29980
for rep in 1 2; do
  for v in old new; do
    cp ab_tmp/_sfgpu_$v.so paper_2102_13018_b200/_sfgpu.so
    for n in 512 1024 2048; do
      p=$((p+1)); timeout 600 $TR --master-port $p bench_configs.py --config 2 --n2 $n --steps 10 > $O/r2ev_${v}_n${n}_r$rep.log 2>&1
    done
  done
done
cp ab_tmp/_sfgpu_new.so paper_2102_13018_b200/_sfgpu.so
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > $O/r2ev_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2ev_tests.log
timeout 400 $TR --master-port 29999 bench.py --gpus 2 > $O/r2ev_bench_n2.log 2>&1
