O=gpurun_out; mkdir -p $O
for c in 1 4; do
  n=8; [ $c = 4 ] && n=16
  timeout 300 python bench_configs.py --config $c --steps 1 --warmup 1 > $O/plain_cfg$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:segments_kernel -c $n -o /tmp/prof_cfg$c python bench_configs.py --config $c --steps 1 --warmup 1 > $O/ncu_cfg$c.log 2>&1
  ncu -i /tmp/prof_cfg$c.ncu-rep --page raw --csv > $O/prof_cfg${c}_raw.csv 2>&1
  ncu -i /tmp/prof_cfg$c.ncu-rep --page source --csv -k regex:segments_kernel --launch-skip 1 --launch-count 1 > $O/prof_cfg${c}_source1.csv 2>&1
done
