# Last check of the committed build: full GPU suite on 4 GPUs, smoke, bench N=1 default, bench N=2
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2j_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2j_tests_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2j_smoke.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2j_bench_n1.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 30111 bench.py --gpus 2 > $O/r2j_bench_n2.log 2>&1
