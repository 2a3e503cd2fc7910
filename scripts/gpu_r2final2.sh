# Final build re-check: full GPU suite on 4 GPUs, smoke, bench N=1/2/4, config 4 at N=1/2/4, config 3 N=4
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2g_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2g_tests_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2g_smoke.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2g_bench_n1.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29871 bench.py --gpus 2 > $O/r2g_bench_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29872 bench.py --gpus 4 > $O/r2g_bench_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench_configs.py --config 4 > $O/r2g_cfg4_n1.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29873 bench_configs.py --config 4 > $O/r2g_cfg4_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29874 bench_configs.py --config 4 > $O/r2g_cfg4_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29875 bench_configs.py --config 3 > $O/r2g_cfg3_n4.log 2>&1
