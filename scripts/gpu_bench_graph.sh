O=gpurun_out; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --no-cpu-baseline --no-e2e --no-device-setup --graph > $O/bg_n1.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 4 --no-e2e --no-device-setup --graph > $O/bg_n4.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29593 bench.py --gpus 4 --no-e2e --no-device-setup > $O/bg_n4_eager.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 2 --no-e2e --no-device-setup --graph > $O/bg_n2.log 2>&1
