O=gpurun_out; mkdir -p $O
timeout 400 python bench_configs.py --config 1 > $O/cfg1_base.log 2>&1

