O=gpurun_out; mkdir -p $O
timeout 300 python bench_configs.py --config 4 --steps 1 --warmup 1 > $O/plain_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr -c 2 -o /tmp/prof_c4 python bench_configs.py --config 4 --steps 1 --warmup 1 > $O/ncu_c4.log 2>&1
ncu -i /tmp/prof_c4.ncu-rep --page raw --csv > $O/prof_c4_raw.csv 2>&1
ncu -i /tmp/prof_c4.ncu-rep --page source --csv --launch-count 1 > $O/prof_c4_source.csv 2>&1
ncu -i /tmp/prof_c4.ncu-rep --page details --csv --launch-count 1 > $O/prof_c4_details.csv 2>&1
