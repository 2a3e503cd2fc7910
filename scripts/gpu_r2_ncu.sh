# Round 2 ncu evidence (one GPU): launch list of the headline bench, full
# captures of its dominant kernels and of the config 1 / config 4 kernels.
O=gpurun_out; mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-device-setup"
$CMD > $O/r2n_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2n_launches_bench.csv $CMD > $O/r2n_ncu_launches.log 2>&1
CMD2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-device-setup"
$CMD2 > $O/r2n_plain_bench2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pair_solo -s 6 -c 2 -o /tmp/r2n_bench $CMD2 > $O/r2n_ncu_bench.log 2>&1
ncu -i /tmp/r2n_bench.ncu-rep --page raw --csv > $O/r2n_bench_raw.csv 2>&1
run() {  # tag regex skip count cmd...
  tag=$1; rx=$2; sk=$3; cnt=$4; shift 4
  "$@" > $O/r2n_plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $sk -c $cnt -o /tmp/r2n_$tag "$@" > $O/r2n_ncu_$tag.log 2>&1
  ncu -i /tmp/r2n_$tag.ncu-rep --page raw --csv > $O/r2n_raw_$tag.csv 2>&1
}
run cfg1 "pair_solo|csr_solo" 0 4 python bench_configs.py --config 1 --steps 1 --warmup 1
run cfg4 "csr_solo|csr_kernel" 0 2 python bench_configs.py --config 4 --steps 1 --warmup 1
