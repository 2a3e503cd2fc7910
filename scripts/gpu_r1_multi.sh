O=gpurun_out; mkdir -p $O
set -x
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench_configs.py --config 5 > $O/cfg5.log 2>&1
timeout 300 python bench_configs.py --config 3 --steps 20 > $O/cfg3.log 2>&1
export CUDA_VISIBLE_DEVICES=0
for c in 1 4; do
  n=8; [ $c = 4 ] && n=24
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:segments_kernel -c $n -o /tmp/prof_cfg$c python bench_configs.py --config $c --steps 1 --warmup 1 > $O/ncu_cfg$c.log 2>&1
  ncu -i /tmp/prof_cfg$c.ncu-rep --page raw --csv > $O/prof_cfg${c}_raw.csv 2>&1
  ncu -i /tmp/prof_cfg$c.ncu-rep --page details --csv > $O/prof_cfg${c}_details.csv 2>&1
  ls -la /tmp/prof_cfg$c.ncu-rep >> $O/ncu_cfg$c.log
done
