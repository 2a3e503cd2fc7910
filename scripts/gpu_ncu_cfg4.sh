O=gpurun_out; mkdir -p $O
timeout 300 python bench_configs.py --config 4 --steps 1 --warmup 1 > $O/plain_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_kernel -c 4 -o /tmp/prof_c4c python bench_configs.py --config 4 --steps 1 --warmup 1 > $O/ncu_c4c.log 2>&1
ncu -i /tmp/prof_c4c.ncu-rep --page raw --csv > $O/prof_c4c_raw.csv 2>&1
