O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/f2_smoke.log 2>&1; echo "rc $?" >> $O/f2_smoke.log
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > $O/f2_gpu_tests.log 2>&1; echo "rc $?" >> $O/f2_gpu_tests.log
timeout 400 python bench.py > $O/f2_bench_n1.log 2>&1
timeout 400 python bench.py --impl reference > $O/f2_bench_ref.log 2>&1
bash profiles/run_ncu.sh $O r1c > $O/f2_ncu.log 2>&1
timeout 300 python bench_configs.py --config 4 --steps 1 --warmup 1 > $O/plain_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr -c 2 -o /tmp/prof_c4b python bench_configs.py --config 4 --steps 1 --warmup 1 > $O/ncu_c4b.log 2>&1
ncu -i /tmp/prof_c4b.ncu-rep --page raw --csv > $O/prof_c4b_raw.csv 2>&1
ncu -i /tmp/prof_c4b.ncu-rep --page details --csv --launch-count 1 > $O/prof_c4b_details.csv 2>&1
