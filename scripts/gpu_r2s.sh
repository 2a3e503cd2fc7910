O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_configs.py --config 3 --spmv > $O/r2s_spmv_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29551 bench_configs.py --config 3 --spmv > $O/r2s_spmv_n2.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x > $O/r2s_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2s_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s_smoke.log 2>&1; echo "rc=$?" >> $O/r2s_smoke.log
