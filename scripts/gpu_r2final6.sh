O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2k_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2k_tests_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2k_smoke.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2k_bench_n1.log 2>&1
