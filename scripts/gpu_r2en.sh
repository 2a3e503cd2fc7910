# SpMV forward + transpose at N=1/2/4; ncu capture of the diagonal SELL kernel
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_configs.py --config 3 --spmv > $O/r2en_spmv_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29881 bench_configs.py --config 3 --spmv > $O/r2en_spmv_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29882 bench_configs.py --config 3 --spmv > $O/r2en_spmv_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_spmv_kernel -s 3 -c 1 -o /tmp/r2en_spmv python bench_configs.py --config 3 --spmv --steps 2 --warmup 1 > $O/r2en_ncu.log 2>&1
ncu -i /tmp/r2en_spmv.ncu-rep --page raw --csv > $O/r2en_spmv_raw.csv 2>&1
