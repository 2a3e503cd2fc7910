O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/v_gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/v_smoke.log 2>&1
timeout 300 python bench.py > $O/v_bench_n1.log 2>&1
timeout 300 python bench.py --impl reference > $O/v_bench_ref.log 2>&1
timeout 300 python bench_configs.py --config 1 --cpu > $O/v_cfg1.log 2>&1
timeout 300 python bench_configs.py --config 4 --cpu > $O/v_cfg4.log 2>&1
bash profiles/run_ncu.sh $O r1b > $O/v_ncu.log 2>&1
