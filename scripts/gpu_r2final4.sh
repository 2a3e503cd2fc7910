# Final build (PDL, one-shot, put chunks, 3-CTA wide exchanges): full GPU suite, smoke, bench N=1/2/4, configs 2/3/4 at N>1
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/r2i_tests_4gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2i_tests_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2i_smoke.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > $O/r2i_bench_n1.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 30061 bench.py --gpus 2 > $O/r2i_bench_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 30062 bench.py --gpus 4 > $O/r2i_bench_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 30063 bench.py --gpus 4 --dims 2,2,1 --no-e2e > $O/r2i_bench_n4_dims221.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 30064 bench_configs.py --config 2 > $O/r2i_cfg2_n4.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 30065 bench_configs.py --config 4 > $O/r2i_cfg4_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 30066 bench_configs.py --config 4 > $O/r2i_cfg4_n4.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 30067 bench_configs.py --config 3 > $O/r2i_cfg3_n4.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 30068 bench_configs.py --config 3 --spmv > $O/r2i_spmv_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 30069 bench_configs.py --config 3 --spmv > $O/r2i_spmv_n4.log 2>&1
