O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/f_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/f_gpu_tests.log 2>&1
timeout 400 python bench.py > $O/f_bench_n1.log 2>&1
timeout 400 python bench.py --impl reference > $O/f_bench_ref.log 2>&1
timeout 300 python scripts/trace_setup.py > $O/f_trace.log 2>&1
