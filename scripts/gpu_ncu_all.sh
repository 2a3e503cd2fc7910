O=gpurun_out; mkdir -p $O
run() {  # tag regex count cmd...
  tag=$1; rx=$2; cnt=$3; shift 3
  "$@" > $O/plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -c $cnt -o /tmp/p_$tag "$@" > $O/ncu_$tag.log 2>&1
  ncu -i /tmp/p_$tag.ncu-rep --page raw --csv > $O/raw_$tag.csv 2>&1
}
run cfg1 "segments_kernel|csr_kernel" 4 python bench_configs.py --config 1 --steps 1 --warmup 1
run cfg4 "csr_kernel" 2 python bench_configs.py --config 4 --steps 1 --warmup 1
run spmv "sell_spmv" 2 python bench_configs.py --config 3 --spmv --steps 1 --warmup 1
