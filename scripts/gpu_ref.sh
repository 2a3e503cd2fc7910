O=gpurun_out; mkdir -p $O
for n in 2 4; do
s=$(date +%s)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --impl reference --gpus $n > $O/ref_n$n.log 2>&1
echo "rc=$? elapsed=$(( $(date +%s) - s )) s" >> $O/ref_n$n.log
done
